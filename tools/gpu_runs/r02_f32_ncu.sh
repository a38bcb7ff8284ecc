set -x
python tools/f32_bench.py > gpurun_out/f32_bench.json 2> gpurun_out/f32_bench.err && \
ncu --set full --clock-control none --import-source on -k regex:k_gather_f32 -c 1 -o /tmp/f32 python tools/f32_bench.py > gpurun_out/ncu_f32.log 2>&1
ncu -i /tmp/f32.ncu-rep --page raw --csv > gpurun_out/r02_ncu_gather_f32_raw.csv 2>&1
ncu -i /tmp/f32.ncu-rep --page source --csv > gpurun_out/r02_ncu_gather_f32_source.csv 2>&1
ls -la gpurun_out
