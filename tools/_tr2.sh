for l in tr_l1 tr_l2 tr_l4 tr_l8; do echo "== $l filter"; IXGPU_LIB=paper_2506_23058_b200/libixgpu_$l.so python tools/trace_filter.py filter 28 | grep -E "span|lookback|life"; done
