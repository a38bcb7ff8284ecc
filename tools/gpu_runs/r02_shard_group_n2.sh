set -x
nvidia-smi -L
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/t2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 tools/sharded_check.py --n 10000000 --queries 1000 > gpurun_out/sc10m_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/b2_n2.json 2> gpurun_out/b2_n2.err
tail -3 gpurun_out/t2.log; tail -3 gpurun_out/sc10m_n2.log; cat gpurun_out/b2_n2.json | head -c 600
