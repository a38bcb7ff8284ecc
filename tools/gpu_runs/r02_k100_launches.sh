# configs[3] k=100, D=350 at HEAD: the launch list (per-kernel device time) of
# one sweep point, to split the step between union and gather.
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_union|k_gather|k_locate|k_qkeys|sort" -c 200 --csv --log-file gpurun_out/k100_launches.csv python tools/sweep.py --depths 350 --curves 8 --ks 100 --recall-sample 100 > gpurun_out/k100_sweep.log 2>&1
