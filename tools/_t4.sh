S='import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],3) for k,v in d.items() if isinstance(v,dict)})'
python tools/kbench.py 28 | python -c "$S"
