set -x
for v in default minb3 b12 minb3b12; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  python tools/sweep.py --depths 350,1024 --curves 8 --ks 10,64,100 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/nu_ab.jsonl
done
unset HCG_LIB_OVERRIDE
cut -c1-160 gpurun_out/nu_ab.jsonl
