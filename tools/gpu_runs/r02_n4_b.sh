# 4-GPU: suite at HEAD, the N=8 per-GPU load proxy (50M over 4 = 12.5M per
# shard at the N=8 planned depth 80), raw-view 10M sharded parity, online
# sweeps at N=1 and N=4 with the fused small-batch kernel, bench N=1 / N=4.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -5 > gpurun_out/t_n4b.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 10 --warmup 3 --rows 50000000 --shard-depth 80 > gpurun_out/b_n4_proxy8.json 2> gpurun_out/b_n4_proxy8.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29562 tools/sharded_check.py --rows 10000000 --queries 1000 --view raw > gpurun_out/sc10m_n4_raw.log 2>&1
timeout 600 python tools/online_sweep.py --gpus 1 > gpurun_out/online_n1.jsonl 2> gpurun_out/online_n1.err
timeout 900 python tools/online_sweep.py --gpus 4 > gpurun_out/online_n4.jsonl 2> gpurun_out/online_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b_n4.json 2> gpurun_out/b_n4.err
python bench.py --steps 10 --warmup 3 > gpurun_out/b_n1.json 2> gpurun_out/b_n1.err
tail -3 gpurun_out/t_n4b.log; grep '^{' gpurun_out/sc10m_n4_raw.log | cut -c1-300
