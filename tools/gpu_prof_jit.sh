# ncu capture of the plan-specialised SHM kernels + lowering variants (JIT)
O=gpurun_out
W=${W:-su2random_n28}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:atlas_shm -s 3 -c 3 -o $O/prof_jit_$W python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > $O/ncu_jit.log 2>&1; tail -2 $O/ncu_jit.log
for opt in "shm_nbuf=2" "shm_rb=3" "shm_nbuf=3" "shm_direct_store=0"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload $W --opt $opt > $O/v.json 2> $O/v.err
  python -c "
import json
d=json.loads(open('$O/v.json').read().strip().splitlines()[-1])
c=d['config']; r=d['roofline']
print('$W $opt', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], c['kernel_ms_per_step'], r['avg_launch_ms'])
" || tail -3 $O/v.err
done
