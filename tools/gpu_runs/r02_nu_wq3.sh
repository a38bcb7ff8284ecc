# Queued union-less walk at every list width (R = 1 / 2 / 4 / 8): parity,
# default dispatch vs the separate union per k and depth, and the N=1 bench.
set -x
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_wq3.log
timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,16,17,32,33,48,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "default", /' > gpurun_out/wq3_ab.jsonl
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so
HCG_NO_UNIONLESS=1 timeout 300 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,17,32,48 --recall-sample 100 | sed 's/^{/{"variant": "union", /' >> gpurun_out/wq3_ab.jsonl
unset HCG_LIB_OVERRIDE
timeout 600 python bench.py > gpurun_out/b_wq3.json 2> gpurun_out/b_wq3.err
cat gpurun_out/t_wq3.log
