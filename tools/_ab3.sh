for lib in "" mb3 mb2; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-default}"; IXGPU_LIB=$L timeout 300 python tools/kbench.py 28 | python tools/kb_short.py
done
