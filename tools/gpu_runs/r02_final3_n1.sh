# Round-end verification at HEAD after the queued union gather, in the
# driver's order: GPU suite, smoke(), reference arm, bench (N=1), the ncu
# launch list of the same bench command and one --set full capture of
# k_gather_nu (reduced to CSV pages on the box); plus the k / depth sweep.
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -6 > gpurun_out/final3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final3_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/final3_reference_arm.json 2> gpurun_out/final3_reference_arm.err
timeout 600 python bench.py > gpurun_out/final3_bench_n1.json 2> gpurun_out/final3_bench_n1.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 > /dev/null 2>&1
mkdir -p /tmp/ncu
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --recall-sample 100 --latency-batches 1 --latency-reps 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_nu -s 3 -c 1 -o /tmp/ncu/gather_nu $CMD > gpurun_out/final3_ncu_full.log 2>&1
ncu -i /tmp/ncu/gather_nu.ncu-rep --page raw --csv > gpurun_out/final3_ncu_gather_nu_raw.csv 2>&1
ncu -i /tmp/ncu/gather_nu.ncu-rep --page details --csv > gpurun_out/final3_ncu_gather_nu_details.csv 2>&1
timeout 400 python tools/sweep.py --depths 128,350,1024 --curves 8 --ks 10,16,17,32,48,64,100,128 --recall-sample 100 | sed 's/^{/{"variant": "final", /' > gpurun_out/final3_sweep.jsonl
cat gpurun_out/final3_gpu_tests.log gpurun_out/final3_smoke.log; cut -c1-300 gpurun_out/final3_reference_arm.json gpurun_out/final3_bench_n1.json
du -sh gpurun_out/final3_*
