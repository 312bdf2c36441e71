# tile / occupancy A/B: default (3 chunks, 4 CTAs) vs 2 chunks with 5 or 6 CTAs per SM
for lib in "" old "" old; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-default}"; IXGPU_LIB=$L timeout 300 python tools/kbench.py 28 | python tools/kb_short.py | tr ' ' '\n' | grep -E "scan_i64|scan_i32|segsum|c2_fused" | tr '\n' ' '; echo
done
