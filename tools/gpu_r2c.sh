# round 2: fused pack + exact staging + parallel kernelize: GPU suite + bench lines
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r2c_gpu_all.log 2>&1; echo "exit $?" >> $O/r2c_gpu_all.log
tail -5 $O/r2c_gpu_all.log
for w in su2random_n28 qsvm_n28; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --workload $w > $O/r2c_$w.json 2> $O/r2c_$w.err
  python -c "
import json
d=json.loads(open('$O/r2c_$w.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$w', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], c['plan']['plan_s'], d['clocks'])
" || tail -3 $O/r2c_$w.err
done
