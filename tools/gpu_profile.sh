#!/bin/bash
# One profiling session for profiles/: parity tests, the default bench line,
# the ncu launch list of the same command and one --set full capture of the
# dominant kernels (the plan-specialised SHM kernels atlas_shm_*, and the
# fused kernel), plus an ising capture.
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 1500 $O/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:atlas_shm -s 13 -c 4 -o $O/prof_shm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_shm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -o $O/prof_fused python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:atlas_shm -s 6 -c 6 -o $O/prof_ising python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload ising_n28 > $O/ncu_ising.log 2>&1
ls $O
