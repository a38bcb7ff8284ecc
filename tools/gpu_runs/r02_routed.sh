# Routed aggregate at N=2 and N=4 (parity of the blocks + bench) and the
# empty-shard group test.
set -x
python -m pytest tests/test_multi_gpu.py tests/test_gpu_parity.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_routed.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29571 tools/sharded_check.py --rows 2000000 --queries 500 > gpurun_out/sc_routed.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b_n4_routed.json 2> gpurun_out/b_n4_routed.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29573 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b_n2_routed.json 2> gpurun_out/b_n2_routed.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29574 bench.py --gpus 4 --steps 10 --warmup 3 --rows 50000000 --shard-depth 80 > gpurun_out/b_n4_proxy8_routed.json 2> gpurun_out/b_n4_proxy8_routed.err
cat gpurun_out/t_routed.log; grep '^{' gpurun_out/sc_routed.log | cut -c1-400
