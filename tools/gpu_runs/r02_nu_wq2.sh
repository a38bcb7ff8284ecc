# Offer queue with the row -> id translation deferred to the flush: parity,
# k > 32 union-less timings, and the same queue for k <= 32 (R = 1, q1 build).
set -x
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_wq2.log
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so
HCG_UNIONLESS_WIDE=1 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,33,64,100,128 --recall-sample 100 | sed 's/^{/{"variant": "wq2", /' > gpurun_out/wq2_ab.jsonl
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-q1/libhcg_q1.so
python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10 --recall-sample 100 | sed 's/^{/{"variant": "q1", /' >> gpurun_out/wq2_ab.jsonl
python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -rf 2>&1 | tail -3 > gpurun_out/t_q1.log
unset HCG_LIB_OVERRIDE
python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10 --recall-sample 100 | sed 's/^{/{"variant": "default", /' >> gpurun_out/wq2_ab.jsonl
cat gpurun_out/t_wq2.log gpurun_out/t_q1.log
