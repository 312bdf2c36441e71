# one GPU session: smoke, every bench config, the reference arm, the C2 launch
# list and ncu --set full captures of the kernels the bench lines name
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
for c in c2 c1 c3 c4 c5; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>&1; echo "launches rc=$?"
for w in c2 filter partition2; do
  timeout 300 python tools/prof_run.py $w 28 2 > /dev/null && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_b -s 1 -c 1 -o gpurun_out/${w}_full python tools/prof_run.py $w 28 2 > /dev/null 2>&1; echo "$w rc=$?"
done
timeout 600 $B --config c3 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scatter_t -c 1 -o gpurun_out/scatter_full $B --config c3 > /dev/null 2>&1; echo "sc rc=$?"
timeout 600 $B --config c4 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_gather -c 1 -o gpurun_out/csr_full $B --config c4 > /dev/null 2>&1; echo "csr rc=$?"
