S='import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],3) for k,v in d.items() if isinstance(v,dict)})'
echo "== default (persistent, lb4)"; python tools/kbench.py 28 | python -c "$S"
echo "== non-persistent lb4"; IXG_PERSIST=0 python tools/kbench.py 28 | python -c "$S"
echo "== persistent lb16"; IXGPU_LIB=paper_2506_23058_b200/libixgpu_lb16.so python tools/kbench.py 28 | python -c "$S"
echo "== non-persistent lb16"; IXG_PERSIST=0 IXGPU_LIB=paper_2506_23058_b200/libixgpu_lb16.so python tools/kbench.py 28 | python -c "$S"
