# HEAD: server tests and the N=1 online sweep (default policy, slots 2).
set -x
timeout 600 python -m pytest tests/test_gpu_server.py -q -p no:cacheprovider -rf 2>&1 | tail -2 > gpurun_out/final3_server_tests.log
timeout 600 python tools/online_sweep.py --gpus 1 > gpurun_out/final3_online_n1.jsonl 2> gpurun_out/final3_online_n1.err
cat gpurun_out/final3_server_tests.log
