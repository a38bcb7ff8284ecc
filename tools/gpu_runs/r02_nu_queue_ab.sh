set -x
python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -rf -k large_batch 2>&1 | tail -3 > gpurun_out/t5.log
for v in default q2 q8 q4m3 knobs; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  if [ $v = knobs ]; then export HCG_NO_UNIONLESS=1; fi
  python tools/sweep.py --depths 128,350,512,1024 --curves 8 --ks 10,64,100,128 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/nuq_ab.jsonl
done
unset HCG_LIB_OVERRIDE HCG_NO_UNIONLESS
cat gpurun_out/t5.log
