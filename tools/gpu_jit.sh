O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
for j in 0 1; do
for w in su2random_n28 qsvm_n28 ising_n28 qft_n28; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload $w --opt shm_jit=$j > $O/it_${w}_$j.json 2> $O/it_${w}_$j.err
  python -c "
import json
d=json.loads(open('$O/it_${w}_$j.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w jit=$j', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], c['plan'].get('jit_s'), c['kernel_ms_per_step'], r['kernel'], r['achieved'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'])
" || tail -3 $O/it_${w}_$j.err
done; done
