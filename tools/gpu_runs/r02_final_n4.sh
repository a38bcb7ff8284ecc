# GPU suite at HEAD on a 4-GPU box (multi-GPU tests included).
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -6 > gpurun_out/final_gpu_tests_n4.log
cat gpurun_out/final_gpu_tests_n4.log
