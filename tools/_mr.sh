# functional check of bench.py's multi-rank path on one GPU (gloo, 2 ranks)
for c in c2 c5; do
  IXG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --config $c --quick > gpurun_out/mr_$c.json 2> gpurun_out/mr_$c.err; echo "$c rc=$?"; tail -c 600 gpurun_out/mr_$c.json
done
