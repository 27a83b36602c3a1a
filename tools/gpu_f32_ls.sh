O=gpurun_out
for w in su2random_n28 qft_n28 ising_n28; do for opt in ls_qubits=4 ls_qubits=5 ls_qubits=6; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --workload $w --dtype f32 --opt $opt > $O/f.json 2> $O/f.err
  python -c "
import json
d=json.loads(open('$O/f.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w f32 $opt', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'])
" || tail -3 $O/f.err
done; done
