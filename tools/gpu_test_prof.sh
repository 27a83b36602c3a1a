O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:atlas_shm -s 3 -c 3 -o $O/prof_jit2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_jit.log 2>&1; tail -1 $O/ncu_jit.log
