# quick GPU loop: parity subset + bench lines (optionally with OPTS)
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${TESTS:+-k "$TESTS"} > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
for w in ${WORKLOADS:-su2random_n28 qsvm_n28 ising_n28 qft_n28}; do
for opt in ${OPTS:-shm_jit=1}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload $w $(for x in ${opt//,/ }; do echo --opt $x; done) > $O/q.json 2> $O/q.err
  python -c "
import json
d=json.loads(open('$O/q.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w $opt', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], c['kernel_ms_per_step'], r['kernel'], r['frac'], r['avg_launch_ms'])
" || tail -3 $O/q.err
done; done
