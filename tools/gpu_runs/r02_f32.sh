# f32 rows at bench scale with the exact sequential sums (round 1 summed in a
# tree: 21.1 ms per 100K queries); parity tests first.
set -x
python -m pytest tests/test_gpu_f32.py tests/test_gpu_fuzz.py tests/test_cpp_wrapper.py -q -p no:cacheprovider -rf -k "f32 or wrapper" 2>&1 | tail -3 > gpurun_out/t_f32.log
python tools/f32_bench.py > gpurun_out/f32_bench.json 2> gpurun_out/f32_bench.err
cat gpurun_out/t_f32.log gpurun_out/f32_bench.json
