# Server: idle batches on one stream (no cross-stream waits); server tests and
# the online sweep at N=1.
set -x
python -m pytest tests/test_gpu_server.py -q -p no:cacheprovider -rf 2>&1 | tail -3 > gpurun_out/t_srv.log
timeout 600 python tools/online_sweep.py --gpus 1 > gpurun_out/online_n1_idle.jsonl 2> gpurun_out/online_n1_idle.err
cat gpurun_out/t_srv.log
python3 -c "
import json
for l in open('gpurun_out/online_n1_idle.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); print(d.get('load',d.get('load_fraction')), round(d.get('throughput_qps',0)/1e6,2), {k:round(v,3) for k,v in d['latency_ms'].items() if k in ('p50','p99')}, round(d['batch_size']['mean'],1))
"
