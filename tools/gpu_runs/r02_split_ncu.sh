set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --recall-sample 100 --latency-batches 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gather_nu -s 3 -c 1 --csv $CMD > gpurun_out/split_ncu.csv 2> gpurun_out/split_ncu.err
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-nosplit/libhcg_nosplit.so ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gather_nu -s 3 -c 1 --csv $CMD > gpurun_out/nosplit_ncu.csv 2>> gpurun_out/split_ncu.err
grep -h "dram__bytes\|gpu__time\|lts__t\|issue_active\|warps_active" gpurun_out/split_ncu.csv gpurun_out/nosplit_ncu.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
