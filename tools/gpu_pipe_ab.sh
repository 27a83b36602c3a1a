O=gpurun_out; mkdir -p $O
for w in su2random_n28 ising_n28 qsvm_n28; do
for p in 1 0; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pab_${w}_$p.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare --workload $w --opt shm_pipe=$p > /dev/null 2>&1; echo "$w pipe=$p exit $?"
done; done
