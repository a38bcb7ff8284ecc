# Locate phase of the small-batch kernel without the lower bound (timing probe
# build) vs the tuning build with it.
set -x
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-knobs/libhcg_knobs.so HCG_SMALL_PROF=1 python tools/small_phases.py > gpurun_out/phases_full.txt 2>&1
HCG_LIB_OVERRIDE=$PWD/paper_1209_0410_b200/csrc/build-nosearch/libhcg_nosearch.so HCG_SMALL_PROF=1 python tools/small_phases.py > gpurun_out/phases_nosearch.txt 2>&1
tail -4 gpurun_out/phases_full.txt gpurun_out/phases_nosearch.txt
