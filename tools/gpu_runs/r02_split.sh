# Two-stage rows in the union-less walk: parity, then bench A/B (release =
# split, MINB 3; nosplit; split at 2 / 4 CTAs per SM).
set -x
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_formats.py -q -p no:cacheprovider -rf -x 2>&1 | tail -4 > gpurun_out/t_split.log
for v in default nosplit splitm2 splitm4 default; do
  if [ $v = default ]; then unset HCG_LIB_OVERRIDE; else export HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cert-sample 100 --recall-sample 200 --latency-batches 1 | python3 -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', d['value'], r['launch_ms'], r['other_kernels_ms'], d['ms_per_step'], d['parity_certificate']['identical'], d['config']['recall_at_k'])" >> gpurun_out/split_ab.txt
done
unset HCG_LIB_OVERRIDE
python bench.py --steps 10 --warmup 3 > gpurun_out/b_split.json 2> gpurun_out/b_split.err
cat gpurun_out/t_split.log gpurun_out/split_ab.txt; python3 -c "import json; d=json.load(open('gpurun_out/b_split.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_vs_reference'])"
