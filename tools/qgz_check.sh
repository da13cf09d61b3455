# qgZ development check on a 4-GPU box: GPU test suite, single-GPU kernel
# microbench, and the per-stage timelines at 1x4, 2x2 and 1x2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_all.log
CUDA_VISIBLE_DEVICES=0 timeout 120 python tools/microbench.py qgz > gpurun_out/mb.log 2>&1
for X in 4 2; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2952$X tools/stage_timeline.py $X > gpurun_out/tl4_$X.log 2> gpurun_out/tl4_$X.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 tools/stage_timeline.py 2 > gpurun_out/tl2_2.log 2> gpurun_out/tl2_2.err
