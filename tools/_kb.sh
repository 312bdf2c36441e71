# GPU tests + per-kernel timings (development loop); each step under its own timeout
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py ${1:-28} > gpurun_out/kbench.json 2>&1
python - <<'PY'
import json
d = json.load(open("gpurun_out/kbench.json"))
print(" ".join(f"{k}={v['ms']:.4f}" for k, v in d.items() if isinstance(v, dict) and "ms" in v))
PY
