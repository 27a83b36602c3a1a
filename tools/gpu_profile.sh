#!/bin/bash
# One profiling session for profiles/: parity tests, the default bench line,
# the ncu launch list of the same command and one --set full capture of the
# dominant kernel (shm_kernel) and of the fused kernel.
O=gpurun_out
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 1500 $O/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shm_kernel -s 30 -c 3 -o $O/prof_shm python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_shm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o $O/prof_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_fused.log 2>&1
ls $O
