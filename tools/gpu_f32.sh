O=gpurun_out
for w in su2random_n28 qft_n28 ghz_n28 su2random_n30; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload $w --dtype f32 > $O/f.json 2> $O/f.err
  python -c "
import json
d=json.loads(open('$O/f.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w f32', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], c['kernel_ms_per_step'], r['frac'], r['avg_launch_ms'])
" || tail -3 $O/f.err
done
