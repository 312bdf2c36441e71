# functional check of the multi-rank bench paths with 4 ranks sharing one GPU (gloo)
for c in c2 c5; do
IXG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 4 --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/dist4_$c.json 2> gpurun_out/dist4_$c.err; echo "$c rc=$?"
tail -1 gpurun_out/dist4_$c.json | cut -c1-400
done
