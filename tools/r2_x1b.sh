O=gpurun_out/x1b; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -k "two_gpus or hop1" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
