# filter/partition bulk-store A/B (IXG_BULK_ALL=1 lib) with a parity run on it
IXGPU_LIB=paper_2506_23058_b200/libixgpu_ba.so timeout 600 python -m pytest tests -q -m gpu -x -k "filter or partition or c2" > gpurun_out/pt_ba.log 2>&1; tail -2 gpurun_out/pt_ba.log
for lib in "" ba "" ba; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-default}"; IXGPU_LIB=$L timeout 300 python tools/kbench.py 28 | python tools/kb_short.py
done
