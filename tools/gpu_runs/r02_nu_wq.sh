# Union-less walk with the warp offer queue (WarpTopK::offer_queued) for k > 32:
# parity (fuzz incl. k <= 128 large batches) and union-less vs union timings.
set -x
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_wq.log
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so
HCG_UNIONLESS_WIDE=1 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,33,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "wq_unionless", /' > gpurun_out/wq_ab.jsonl
HCG_NO_UNIONLESS=1 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 33,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "union", /' >> gpurun_out/wq_ab.jsonl
unset HCG_LIB_OVERRIDE
cat gpurun_out/t_wq.log
