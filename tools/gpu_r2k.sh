# round 2 final profile session (autotuned build): default bench line, launch list of the same command,
# ncu --set full of every SHM launch of one su2random n=28 run, other families
O=gpurun_out; mkdir -p $O
nproc > $O/r2k_host.txt; lscpu | grep -i "model name" >> $O/r2k_host.txt; free -g | head -2 >> $O/r2k_host.txt
timeout 900 python bench.py > $O/r2k_bench_default.json 2> $O/r2k_bench_default.err; tail -c 3000 $O/r2k_bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2k_launches.csv python bench.py --steps 2 --warmup 5 --no-e2e --no-cpu --no-compare > $O/r2k_launches_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:atlas_shm -s 55 -c 11 -o $O/r2k_su2 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu --no-compare > $O/r2k_ncu.log 2>&1
for w in qft_n28 ghz_n28 graphstate_n28 qsvm_n28 wstate_n28 ising_n28; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --workload $w > $O/r2k_$w.json 2> $O/r2k_$w.err
  python -c "
import json
d=json.loads(open('$O/r2k_$w.json').read().strip().splitlines()[-1])
c=d.get('details', d['config']); r=d['roofline']
print('$w', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'])
" || tail -3 $O/r2k_$w.err
done
for w in su2random_n28 qft_n28; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --workload $w --dtype f32 > $O/r2k_${w}_f32.json 2> $O/r2k_${w}_f32.err
  python -c "
import json
d=json.loads(open('$O/r2k_${w}_f32.json').read().strip().splitlines()[-1])
c=d.get('details', d['config']); r=d['roofline']
print('$w f32', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'])
" || tail -3 $O/r2k_${w}_f32.err
done
for w in su2random_n33 qft_n33; do
  timeout 600 python bench.py --steps 3 --warmup 5 --no-e2e --no-cpu --workload $w > $O/r2k_$w.json 2> $O/r2k_$w.err
  python -c "
import json
d=json.loads(open('$O/r2k_$w.json').read().strip().splitlines()[-1])
c=d.get('details', d['config']); r=d['roofline']
print('$w', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'])
" || tail -3 $O/r2k_$w.err
done
