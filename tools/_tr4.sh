python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for w in filter c2; do echo "== $w"; IXGPU_LIB=paper_2506_23058_b200/libixgpu_tr.so python tools/trace_filter.py $w 28; done
S='import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],3) for k,v in d.items() if isinstance(v,dict)})'
python tools/kbench.py 28 | python -c "$S"
