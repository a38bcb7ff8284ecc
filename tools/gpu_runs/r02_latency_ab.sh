# Same-box interleaved latency A/B: the library before the offer-queue work
# (old, commit f266418) vs HEAD (default), three repetitions each.
set -x
for rep in 1 2 3; do
for v in old default; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  timeout 300 python tools/latency_probe.py | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/lat_ab.jsonl
done
done
