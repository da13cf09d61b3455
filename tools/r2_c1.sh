O=gpurun_out/c1b; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_comm_single.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python tools/config1_probe.py > $O/config1.txt 2>&1
for c in c1q c1d k3 k2; do timeout 120 python tools/profile_kernels.py $c 20 >> $O/kernels.jsonl 2>&1; done
