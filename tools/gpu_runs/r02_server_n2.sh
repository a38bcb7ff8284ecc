set -x
python -m pytest tests/test_gpu_server.py tests/test_multi_gpu.py tests/test_gpu_f32.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/t3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 tools/sharded_check.py --rows 10000000 --queries 1000 > gpurun_out/sc10m_n2.log 2>&1
timeout 600 python tools/online_sweep.py --gpus 1 > gpurun_out/online_n1.jsonl 2> gpurun_out/online_n1.err
timeout 900 python tools/online_sweep.py --gpus 2 > gpurun_out/online_n2.jsonl 2> gpurun_out/online_n2.err
tail -3 gpurun_out/t3.log; tail -3 gpurun_out/sc10m_n2.log; cut -c1-400 gpurun_out/online_n*.jsonl; tail -5 gpurun_out/online_n*.err
