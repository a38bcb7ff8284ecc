# Single-process shard group: the fused exchange (search kernels store their
# packed top-k into GPU 0 over NVLink) vs NCCL all-gather (tuning build,
# HCG_SHARD_NCCL=1): correctness (C++ test, server test) and the online
# sweep at N=4; then the GPU suite under the bounds-checked build.
set -x
python -m pytest tests/test_multi_gpu.py tests/test_gpu_server.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_p2p.log
timeout 900 python tools/online_sweep.py --gpus 4 --loads 0.05,0.2,0.6,1.0 > gpurun_out/online_n4_p2p.jsonl 2> gpurun_out/online_n4_p2p.err
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_SHARD_NCCL=1 timeout 900 python tools/online_sweep.py --gpus 4 --loads 0.05,0.2,0.6,1.0 > gpurun_out/online_n4_nccl.jsonl 2> gpurun_out/online_n4_nccl.err
timeout 1500 bash tools/debug_bounds.sh > gpurun_out/debug_bounds.log 2>&1; tail -3 gpurun_out/debug_bounds.log
cat gpurun_out/t_p2p.log
