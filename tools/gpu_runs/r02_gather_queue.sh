# The union path's gather (k_gather) with the offer queue (default) vs the
# per-pass offers (noq): parity suites at HEAD, then a same-box interleaved
# A/B on the union path (HCG_NO_UNIONLESS), twice.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf -x 2>&1 | tail -4 > gpurun_out/t_gq.log
export HCG_NO_UNIONLESS=1
for rep in 1 2; do
for v in noq knobs; do
  export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so
  timeout 300 python tools/sweep.py --depths 128,350 --curves 8 --ks 10,32,64,100 --recall-sample 100 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> gpurun_out/gather_queue_ab.jsonl
done
done
cat gpurun_out/t_gq.log
