# Same-box A/B of the k <= 32 union-less walk: the previous commit's one-at-a-time
# inserts (old), the queued R = 1 list (default, k <= 16), the queued R = 2 list
# for every k <= 48 (r2k10); interleaved, twice.
set -x
for rep in 1 2; do
for v in old default r2k10; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  timeout 300 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,16 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/nu_ab_final.jsonl
done
done
