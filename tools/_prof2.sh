set -x
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
python tools/prof_run.py filter 28 2 && ncu --set full --clock-control none --import-source on -k regex:k_filter_p -s 1 -c 1 -o gpurun_out/filter_p python tools/prof_run.py filter 28 2 > gpurun_out/ncu1.log 2>&1
python tools/prof_run.py partition2 28 2 && ncu --set full --clock-control none --import-source on -k regex:k_place_p -s 1 -c 1 -o gpurun_out/place_p python tools/prof_run.py partition2 28 2 > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu1.log; tail -2 gpurun_out/ncu2.log
