python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
S='import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],3) for k,v in d.items() if isinstance(v,dict)})'
python tools/kbench.py 28 | python -c "$S"
IXG_BIG=0 python tools/kbench.py 28 | python -c "$S"
