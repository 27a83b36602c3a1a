# E6-style ablation: Kernelize vs OrderedKernelize vs greedy-5 fusion vs front packing,
# measured ms/step and kernel counts at n=28 fp64 (one GPU).
O=gpurun_out
echo "| family | kernelizer | kernels (fused/shm) | ms/step | amp-updates/s |" > $O/ablation.md
echo "|---|---|---|---|---|" >> $O/ablation.md
for w in su2random_n28 qft_n28 ising_n28 qsvm_n28 ghz_n28 wstate_n28 graphstate_n28; do
for k in 0 1 2 3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --workload $w --kernelizer $k > $O/ab.json 2> $O/ab.err
  python -c "
import json
names={0:'Kernelize',1:'OrderedKernelize',2:'greedy-5 fusion',3:'front packing'}
d=json.loads(open('$O/ab.json').read().strip().splitlines()[-1])
p=d['config']['plan']
print('| $w | %s | %d (%d/%d) | %.3f | %.3g |' % (names[$k], p['kernels'], p['fusion_kernels'], p['shm_kernels'], d['ms_per_step'], d['value']))
" >> $O/ablation.md || (echo "| $w | $k | failed | | |" >> $O/ablation.md; tail -3 $O/ab.err)
done; done
cat $O/ablation.md
