set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --cert-sample 0 --recall-sample 100 --latency-batches 1"
M=dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
for g in 32 64 128; do
  for v in knobs nosplitk; do
    HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so HCG_L2_FETCH=$g $CMD > gpurun_out/plain_$v_$g.log 2>&1
    HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-$v/libhcg_$v.so HCG_L2_FETCH=$g ncu --metrics $M --clock-control none -k regex:k_gather_nu -s 3 -c 1 --csv $CMD 2>/dev/null | grep '^"0"' | sed "s/^/$v gran=$g /" >> gpurun_out/gran.csv
  done
done
cut -d, -f1,13-15 gpurun_out/gran.csv
