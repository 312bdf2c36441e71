S='import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],3) for k,v in d.items() if isinstance(v,dict) and k in ("c2_fused_kernel","filter_kernel","place_kernel","scan_i64","c2_elided")})'
for lib in s8_l1 s8_l4 s16_l2 s1_l1; do
 for pm in 0 1; do
  echo "== $lib persist=$pm"; IXG_PERSIST=$pm IXGPU_LIB=paper_2506_23058_b200/libixgpu_$lib.so python tools/kbench.py 28 | python -c "$S"
 done
done
