for w in ${@:-filter c2}; do echo "== big $w"; IXGPU_LIB=paper_2506_23058_b200/libixgpu_tr.so timeout 300 python tools/trace_filter.py $w 28; done
