# Server: side-by-side small batches + pipeline stages (pick); server tests and
# sweep at N=1 with 2 and 4 slots.
set -x
python -m pytest tests/test_gpu_server.py -q -p no:cacheprovider -rf 2>&1 | tail -3 > gpurun_out/t_srv.log
for S in 2 4; do
timeout 600 python tools/online_sweep.py --gpus 1 --slots $S > gpurun_out/online_n1_pick_s$S.jsonl 2> gpurun_out/online_n1_pick_s$S.err
done
cat gpurun_out/t_srv.log
for S in 2 4; do echo slots $S; python3 -c "
import json,sys
for l in open(sys.argv[1]):
    if not l.startswith('{'): continue
    d=json.loads(l); print(d.get('load',d.get('load_fraction')), round(d.get('throughput_qps',0)/1e6,2), {k:round(v,3) for k,v in d['latency_ms'].items() if k in ('p50','p99')}, round(d['batch_size']['mean'],1))
" gpurun_out/online_n1_pick_s$S.jsonl; done
