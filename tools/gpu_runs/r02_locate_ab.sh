# k_locate min-blocks A/B (8 = release: 64 registers + an 80-B stack frame;
# 6 / 4: more registers) on the bench workload, then smoke() at HEAD.
set -x
for v in default loc6 loc4; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  for i in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cert-sample 0 --recall-sample 100 --latency-batches 1 | python3 -c "import json,sys; d=json.load(sys.stdin); print('$v', d['value'], d['roofline']['other_kernels_ms'], d['roofline']['launch_ms'], d['ms_per_step'])" >> gpurun_out/locate_ab.txt
  done
done
unset HCG_LIB_OVERRIDE
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
cat gpurun_out/locate_ab.txt gpurun_out/smoke.log
