# round 2: dense hoisting + in-place remap tests + A/B bench
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r2e_gpu_all.log 2>&1; echo "exit $?" >> $O/r2e_gpu_all.log
tail -3 $O/r2e_gpu_all.log
for w in su2random_n28 qsvm_n28 ising_n28; do
for opt in shm_hoist_dense=1 shm_hoist_dense=0; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --workload $w --opt $opt > $O/v.json 2> $O/v.err
  python -c "
import json
d=json.loads(open('$O/v.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w $opt', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'])
" || tail -3 $O/v.err
done; done
