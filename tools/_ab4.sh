# C2 bulk-store A/B: parity on the new default, then kbench default vs IXG_BULK_ST=0
timeout 600 python -m pytest tests -q -m gpu -x -k "c2 or C2 or filter" > gpurun_out/pt_c2.log 2>&1; tail -2 gpurun_out/pt_c2.log
for lib in "" nb "" nb; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-bulk}"; IXGPU_LIB=$L timeout 300 python tools/kbench.py 28 | python tools/kb_short.py
done
