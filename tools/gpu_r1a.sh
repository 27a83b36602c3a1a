#!/bin/bash
# one GPU session: tests, bench lines, launch list, ncu full capture
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in qft_n28 ghz_n28 ising_n28 graphstate_n28 qsvm_n28 wstate_n28; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload su2random_n28 --kernelizer 1 > $O/bench_su2_ok.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --workload su2random_n28 --kernelizer 2 > $O/bench_su2_greedy.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shm_kernel -s 10 -c 2 -o $O/prof_shm python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_shm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 4 -c 2 -o $O/prof_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --workload su2random_n28 --kernelizer 2 > $O/ncu_fused.log 2>&1
ls -la $O
