# HEAD with the queued union gather (R = 1 / 4 / 8) and the new dispatch
# thresholds: parity suites, then the k / depth sweep under default dispatch.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/t_gq3.log
timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,16,17,32,33,48,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "default", /' > gpurun_out/gq3_sweep.jsonl
cat gpurun_out/t_gq3.log
