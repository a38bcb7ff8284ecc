# HEAD on a 4-GPU box: the GPU suite (multi-GPU tests included), then the
# sharded bench at N=2 and N=4 (configs[2], 100M rows, routed aggregate).
set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -6 > gpurun_out/final3_gpu_tests_n4.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/final3_bench_n$N.json 2> gpurun_out/final3_bench_n$N.err
done
cat gpurun_out/final3_gpu_tests_n4.log; cut -c1-300 gpurun_out/final3_bench_n2.json gpurun_out/final3_bench_n4.json
