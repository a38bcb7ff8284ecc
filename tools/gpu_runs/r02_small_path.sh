set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/t6.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b6.json 2> gpurun_out/b6.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --latency-batches 1,4,16,64,256,512,1024 --latency-reps 50 > gpurun_out/lat_default.json 2>/dev/null
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_NO_SMALL=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --latency-batches 1,4,16,64,256,512,1024 --latency-reps 50 > gpurun_out/lat_nosmall.json 2>/dev/null
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_UNIONLESS_WIDE=1 python tools/sweep.py --depths 350,1024 --curves 8 --ks 64,100 --recall-sample 100 | sed 's/^{/{"variant": "unionless_wide", /' > gpurun_out/k_ab.jsonl
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_NO_UNIONLESS=1 python tools/sweep.py --depths 350,1024 --curves 8 --ks 64,100 --recall-sample 100 | sed 's/^{/{"variant": "union", /' >> gpurun_out/k_ab.jsonl
tail -3 gpurun_out/t6.log
