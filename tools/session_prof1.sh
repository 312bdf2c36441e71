set -x
export PYTHONPATH=$PWD
CHECKED=1 python tools/prof_run.py c2 28 3 && CHECKED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_run.py c2 28 2 > gpurun_out/ncu_c2_checked.csv 2> gpurun_out/ncu_c2_checked.err
CHECKED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_run.py partition2 28 2 > gpurun_out/ncu_p2_checked.csv 2>> gpurun_out/ncu_c2_checked.err
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -2 gpurun_out/*.err
