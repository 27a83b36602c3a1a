# round 2, first GPU check: the pipe-mode mbarrier fix against the new
# full-state / grid-capped parity tests, then the whole GPU suite and a bench line
O=gpurun_out; mkdir -p $O
nproc > $O/host_nproc.txt; lscpu | grep -i "model name" >> $O/host_nproc.txt
timeout 900 python -m pytest tests/test_gpu_fullstate.py -q -x > $O/r2a_fullstate.log 2>&1; echo "exit $?" >> $O/r2a_fullstate.log
tail -5 $O/r2a_fullstate.log
timeout 1500 python -m pytest tests -m gpu -q > $O/r2a_gpu_all.log 2>&1; echo "exit $?" >> $O/r2a_gpu_all.log
tail -8 $O/r2a_gpu_all.log
for w in su2random_n28 qsvm_n28 ising_n28 qft_n28; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --workload $w > $O/r2a_$w.json 2> $O/r2a_$w.err
  python -c "
import json
d=json.loads(open('$O/r2a_$w.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks'])
" || tail -3 $O/r2a_$w.err
done
