# bench.py --gpus 2 with both ranks on the one GPU (gloo): the N>1 code path end to end, layer EP over
# IPC-mapped peer memory, then expert-parallel serving on the LockstepClock (numbers are NOT scaling numbers)
mkdir -p gpurun_out
QMOE_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --serve-duration 15 --serve-kv-gib 8 --serve-schedulers baseline,qllm > gpurun_out/bench_ep2.log 2> gpurun_out/bench_ep2.err
echo "exit $?" >> gpurun_out/bench_ep2.log
tail -c 2500 gpurun_out/bench_ep2.log; tail -n 5 gpurun_out/bench_ep2.err
