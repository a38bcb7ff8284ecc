# 4-GPU evidence: GPU suite, 10M sharded parity vs the reference TUs, configs[2]
# at N=4 (100M), the N=8 per-GPU load proxy (50M over 4 = 12.5M per shard at
# the N=8 planned depth 80), and the online sweep over a 4-GPU shard group.
set -x
nvidia-smi -L
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -8 > gpurun_out/t_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29551 tools/sharded_check.py --rows 10000000 --queries 1000 > gpurun_out/sc10m_n4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b_n4.json 2> gpurun_out/b_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29553 bench.py --gpus 4 --steps 10 --warmup 3 --rows 50000000 --shard-depth 80 > gpurun_out/b_n4_proxy8.json 2> gpurun_out/b_n4_proxy8.err
timeout 900 python tools/online_sweep.py --gpus 4 > gpurun_out/online_n4.jsonl 2> gpurun_out/online_n4.err
tail -3 gpurun_out/t_n4.log; grep '^{' gpurun_out/sc10m_n4.log | cut -c1-300
python tools/latency_probe.py > gpurun_out/latency_probe_v2.jsonl 2> gpurun_out/latency_probe_v2.err
cat gpurun_out/latency_probe_v2.jsonl
