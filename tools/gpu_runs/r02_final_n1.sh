# Round-end verification in the driver's order on one B200 at HEAD:
# GPU suite, smoke(), reference arm, bench (N=1), then the ncu launch list of
# the same bench command.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -6 > gpurun_out/final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
python bench.py --impl reference > gpurun_out/final_reference_arm.json 2> gpurun_out/final_reference_arm.err
python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 > /dev/null 2>&1
cat gpurun_out/final_gpu_tests.log gpurun_out/final_smoke.log; cut -c1-400 gpurun_out/final_reference_arm.json gpurun_out/final_bench_n1.json
