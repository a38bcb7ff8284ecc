mkdir -p gpurun_out
for k in 50 64; do for e in "" "HCG_NU_R2=1" "" "HCG_NU_R2=1"; do
  env $e timeout 300 python bench.py --k $k --steps 10 --warmup 3 --cpu-sample 2000 --latency-batches 1 --latency-reps 2 --recall-sample 200 2>gpurun_out/r2_err.txt | python -c "
import json,sys
b=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('k=$k $e', b['value'], b['ms_per_step'], b['config']['recall_at_k'], b.get('parity_vs_reference'))" >> gpurun_out/nu_r2.txt 2>&1
done; done
cat gpurun_out/nu_r2.txt
