# round 2: in-place remap fix + offload tier tests + whole GPU suite
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullstate.py -q -k "inplace or offload" > $O/r2f_new.log 2>&1; echo "exit $?" >> $O/r2f_new.log
tail -15 $O/r2f_new.log
timeout 1500 python -m pytest tests -m gpu -q > $O/r2f_gpu_all.log 2>&1; echo "exit $?" >> $O/r2f_gpu_all.log
tail -6 $O/r2f_gpu_all.log
