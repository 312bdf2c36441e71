# C2 bench step (ms) and CHECKED step with two library builds
for lib in "" old "" old; do
  if [ -z "$lib" ]; then L=paper_2506_23058_b200/libixgpu.so; else L=paper_2506_23058_b200/libixgpu_$lib.so; fi
  echo "== ${lib:-default} $(IXGPU_LIB=$L timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["checked"]["ms_per_step"])')"
done
