# The N > 1 bench path (sharded presence build, stripe render, gather) with two gloo ranks sharing
# one GPU (dev tool; the numbers are not a scaling measurement).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
VSB200_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu \
  > gpurun_out/ws2_gloo.json 2> gpurun_out/ws2_gloo.err
echo "exit $?" >> gpurun_out/ws2_gloo.err
