# Small-batch latency: GPU suite (parity of every path), phase stamps of the
# one-CTA-per-query kernel (tuning build), host/device latency per batch size.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -5 > gpurun_out/t_lat.log
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_SMALL_PROF=1 python tools/small_phases.py > gpurun_out/small_phases.txt 2>&1
python tools/latency_probe.py > gpurun_out/latency_probe.jsonl 2> gpurun_out/latency_probe.err
cat gpurun_out/t_lat.log; tail -4 gpurun_out/small_phases.txt; cat gpurun_out/latency_probe.jsonl
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --cert-sample 50 --latency-batches 1,16,64,128,256,4096,65536 --latency-reps 50 > gpurun_out/b_lat.json 2> gpurun_out/b_lat.err
python3 -c "import json; d=json.load(open('gpurun_out/b_lat.json')); print(d['value'], {k:(v['p50_ms'],v['p99_ms']) for k,v in d['latency'].items()})"
