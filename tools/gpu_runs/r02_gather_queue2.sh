# With the queued union-path gather: union-less (HCG_UNIONLESS_WIDE) vs union
# (HCG_NO_UNIONLESS) per k and depth, to set the dispatch thresholds; and the
# queue-less union gather (noq) at k = 17..64.
set -x
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so
HCG_UNIONLESS_WIDE=1 timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,17,32,48,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "unionless", /' > gpurun_out/gq2.jsonl
HCG_NO_UNIONLESS=1 timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,17,32,48,64,100,112,128 --recall-sample 100 | sed 's/^{/{"variant": "union_queued", /' >> gpurun_out/gq2.jsonl
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-noq/libhcg_noq.so
HCG_NO_UNIONLESS=1 timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 17,32,48,64 --recall-sample 100 | sed 's/^{/{"variant": "union_noq", /' >> gpurun_out/gq2.jsonl
