# Small-batch kernel: rolled (compact) vs unrolled key transform: phase stamps
# (tuning builds) and latency of the release build.
set -x
for v in knobs unrolledkey; do
  HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so HCG_SMALL_PROF=1 python tools/small_phases.py 2>&1 | tail -n 4 | sed "s/^/$v /" >> gpurun_out/phases_key.txt
done
python tools/latency_probe.py > gpurun_out/latency_probe_key.jsonl 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x -k "batch_size or parity" 2>&1 | tail -2
cat gpurun_out/phases_key.txt gpurun_out/latency_probe_key.jsonl
