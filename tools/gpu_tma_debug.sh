O=gpurun_out; mkdir -p $O
for w in su2random qsvm ising qft; do timeout 120 python tools/tma_perf.py $w 28 20 - shm_tma=0 - shm_tma=0; done
