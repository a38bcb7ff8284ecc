# Same-box interleaved A/B, three repetitions: the committed HEAD (prev: union
# gather with per-pass offers, old thresholds) vs the queued union gather with
# the new thresholds (cur), default dispatch, k = 10 ... 128 at D = 128 / 350.
set -x
for rep in 1 2 3; do
for v in prev cur; do
  export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so
  timeout 300 python tools/sweep.py --depths 128,350 --curves 8 --ks 10,32,33,48,64,100,128 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/gq4.jsonl
done
done
