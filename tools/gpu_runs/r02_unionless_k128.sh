set -x
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -p no:cacheprovider -rf 2>&1 | tail -8 > gpurun_out/t4.log
python tools/sweep.py --depths 350,1024 --curves 8 --ks 10,33,64,96,100,128 > gpurun_out/sweep_nu.jsonl 2> gpurun_out/sweep_nu.err
HCG_NO_UNIONLESS=1 python tools/sweep.py --depths 350,1024 --curves 8 --ks 33,64,96,100,128 > gpurun_out/sweep_union.jsonl 2> gpurun_out/sweep_union.err
python bench.py --k 100 --steps 5 --warmup 3 --latency-batches 1 > gpurun_out/b_k100.json 2> gpurun_out/b_k100.err
cat gpurun_out/t4.log; cut -c1-200 gpurun_out/sweep_*.jsonl
