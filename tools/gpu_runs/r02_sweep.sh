# configs[3] at HEAD: depth x curves x k sweep on 10M lifted rows, 100K queries.
set -x
timeout 2400 python tools/sweep.py --depths 16,64,128,256,350,512,1024,4096 --curves 2,4,8,16 --ks 10,100 --recall-sample 500 > gpurun_out/sweep_r02.jsonl 2> gpurun_out/sweep_r02.err
wc -l gpurun_out/sweep_r02.jsonl; tail -2 gpurun_out/sweep_r02.err
