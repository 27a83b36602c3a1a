O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "n33" > $O/pytest_n33.log 2>&1; tail -3 $O/pytest_n33.log
for w in qft_n33 ghz_n33 su2random_n33; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --workload $w > $O/q33.json 2> $O/q33.err
  python -c "
import json
d=json.loads(open('$O/q33.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w', d['ms_per_step'], '%.3g'%d['value'], c['plan'], c['kernel_ms_per_step'], r['frac'], r['avg_launch_ms'])
" || tail -3 $O/q33.err
done
