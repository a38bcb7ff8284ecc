# Offer-queue union-less walk: min-blocks 2 (default) vs 3 for the R = 4 / 8 lists.
set -x
for v in knobs m3; do
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so
HCG_UNIONLESS_WIDE=1 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 33,64,100,128 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/wq_m3.jsonl
done
