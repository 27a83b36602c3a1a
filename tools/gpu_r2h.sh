# round 2 (re-entry): whole GPU suite at HEAD, then the profile session (gpu_r2g.sh)
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/r2h_gpu_all.log 2>&1; echo "exit $?" >> $O/r2h_gpu_all.log
tail -8 $O/r2h_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2h_smoke.log 2>&1; echo "smoke exit $?"; tail -3 $O/r2h_smoke.log
bash tools/gpu_r2g.sh
