#!/bin/bash
# 2-process gloo runs on one GPU, repeated, with a stack dump on a hang
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
  for c in c2 c5; do
    IXG_HANG_DUMP=100 IXG_DIST_BACKEND=gloo timeout 150 python bench.py --gpus 2 --config $c --quick --steps 3 --warmup 3 > gpurun_out/r2_${c}_$i.json 2> gpurun_out/r2_${c}_$i.err
    echo "$c run $i rc=$?"
  done
done
