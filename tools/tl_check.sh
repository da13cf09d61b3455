# per-stage timelines at 1x4 / 2x2 (4 GPUs) and 1x2 (2 GPUs), plus the multi-GPU parity tests
O=${OUT:-gpurun_out}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_comm_single.py tests/test_gpu_collectives.py tests/test_gpu_codec.py -q -x > $O/t_dist.log 2>&1; echo "tests rc=$?" >> $O/t_dist.log
for X in 4 2; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2952$X tools/stage_timeline.py $X > $O/tl4_$X.log 2> $O/tl4_$X.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 tools/stage_timeline.py 2 > $O/tl2_2.log 2> $O/tl2_2.err
