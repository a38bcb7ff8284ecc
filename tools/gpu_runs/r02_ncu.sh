# ncu evidence for round 2 (one tool per call): the launch list of a short
# bench run, the --set full capture of the dominant kernel (k_gather_nu) and
# of the small-batch kernel; plus the latency probe and the gather
# micro-benchmark (LDG / LDGSTS / cp.async.bulk / TMA gather4) without ncu.
# The .ncu-rep files are reduced to CSV pages on the box (gpurun_out <= 64 MiB).
set -x
python tools/latency_probe.py > gpurun_out/latency_probe.jsonl 2> gpurun_out/latency_probe.err
./tools/gather_bench > gpurun_out/gather_bench.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --recall-sample 100 --latency-batches 1,16,64,128 --latency-reps 3"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv $CMD > /dev/null 2>&1
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_gather_nu -s 3 -c 1 -o /tmp/ncu/gather_nu $CMD > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_search_small -s 2 -c 2 -o /tmp/ncu/search_small $CMD > gpurun_out/ncu_full2.log 2>&1
for r in gather_nu search_small; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/r02_ncu_${r}_raw.csv 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/r02_ncu_${r}_details.csv 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv > gpurun_out/r02_ncu_${r}_source.csv 2>&1
done
du -sh gpurun_out/*
