# C1 (2^20 partition2, latency-bound) with alternative builds (wider look-back windows, smaller tiles)
for lib in "" ch1 ch2 "" ch1 ch2; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-default} $(IXGPU_LIB=$L timeout 300 python bench.py --config c1 --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["value"])')"
done
