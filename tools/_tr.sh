for l in trace trace256; do for w in filter c2; do echo "== $l $w"; IXGPU_LIB=paper_2506_23058_b200/libixgpu_$l.so python tools/trace_filter.py $w 28; done; done
