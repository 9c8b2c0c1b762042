# round-2 (session 5): the bench launched through torch.distributed.run with one rank (the sharded entry point + NCCL plane of size 1)
set -x
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r61_torchrun_1rank.json 2> gpurun_out/r61_torchrun.err; echo "rc=$?"
cut -c1-900 gpurun_out/r61_torchrun_1rank.json; tail -3 gpurun_out/r61_torchrun.err
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | tail -3
