mkdir -p gpurun_out
for v in "3 0" "2 0" "4 0" "3 2" "4 3" "3 0" "2 0" "4 0"; do
  set -- $v
  HCG_NU_MINB=$1 HCG_NU_PER_SM=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --latency-batches 1 --latency-reps 2 --recall-sample 100 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=b['roofline']
print('minb=$1 cap=$2', b['value'], r['launch_ms'], r['frac'], b.get('parity_vs_reference'))" >> gpurun_out/nu_ab.txt 2>&1
done
cat gpurun_out/nu_ab.txt
