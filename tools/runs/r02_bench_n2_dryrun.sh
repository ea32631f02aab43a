# Dry run of bench.py's N > 1 path on a one-GPU box: two ranks on cuda:0, gloo
# plumbing (timing meaningless; checks the sharded code path end to end)
PS_BENCH_DEVICE=0 PS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-compare --no-c5 \
    --no-e2e --no-cpu-baseline > gpurun_out/bench_n2_dryrun.log 2> gpurun_out/bench_n2_dryrun.err
echo rc=$?; tail -c 1500 gpurun_out/bench_n2_dryrun.log; tail -5 gpurun_out/bench_n2_dryrun.err
