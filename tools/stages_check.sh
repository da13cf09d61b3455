# qgZ stage sweep + per-stage timelines on a 4-GPU box (for the alpha-beta
# comparison in DESIGN.md), and the qwZ/qgZ timelines at 1x4, 2x2, 1x2.
mkdir -p gpurun_out
for X in 4 2; do
  ZPP_BENCH_SECTIONS=qgz ZPP_BENCH_STAGES=1,2,4,8 timeout 300 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961$X tools/bench_zeropp.py $X > gpurun_out/sweep4_$X.json 2> gpurun_out/sweep4_$X.err
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2952$X tools/stage_timeline.py $X > gpurun_out/tl4_$X.log 2> gpurun_out/tl4_$X.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 tools/stage_timeline.py 2 > gpurun_out/tl2_2.log 2> gpurun_out/tl2_2.err
