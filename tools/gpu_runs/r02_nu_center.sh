# Union-less walk order: each window from its middle outwards (center build)
# vs start to end (default): fuzz parity of the center build, then a same-box
# interleaved A/B, twice.
set -x
export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-center/libhcg_center.so
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -rf -x 2>&1 | tail -4 > gpurun_out/t_center.log
for rep in 1 2; do
for v in default center; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  timeout 300 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,32,100 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/nu_center.jsonl
done
done
cat gpurun_out/t_center.log
