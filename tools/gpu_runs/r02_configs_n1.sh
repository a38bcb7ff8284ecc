# One-GPU configuration evidence: raw view at configs[1] (parity over all 100K
# queries vs the reference TUs), configs[0] (1M x 10K, the whole CPU run
# beside), configs[2] at N=1 (100M on one B200: D=350 and the per-shard
# depths 226 / 134 / 80 of N=2 / 4 / 8), and the reference arm at 100K
# queries per step (same config as the GPU arm); small-batch phase times.
set -x
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_SMALL_PROF=1 python tools/small_phases.py > gpurun_out/small_phases.txt 2>&1
python bench.py --view raw --steps 10 --warmup 3 > gpurun_out/b_raw.json 2> gpurun_out/b_raw.err
python bench.py --rows 1000000 --queries 10000 --cpu-sample 10000 --steps 10 --warmup 3 > gpurun_out/b_c0.json 2> gpurun_out/b_c0.err
for D in 350 226 134 80; do
  python bench.py --rows 100000000 --depth $D --steps 5 --warmup 3 --latency-batches 1,4096 > gpurun_out/b_c2n1_d$D.json 2> gpurun_out/b_c2n1_d$D.err
done
time python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err
cut -c1-300 gpurun_out/b_*.json gpurun_out/ref_arm.json; tail -5 gpurun_out/small_phases.txt
