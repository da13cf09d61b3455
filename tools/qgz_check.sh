# qgZ development check on a 4-GPU box: GPU test suite, single-GPU kernel
# microbench (product tables on / off), and the per-stage timelines at 1x4,
# 2x2 and 1x2.   OUT=gpurun_out/x bash tools/qgz_check.sh
O=${OUT:-gpurun_out}; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/t_all.log 2>&1; echo "tests rc=$?" >> $O/t_all.log
CUDA_VISIBLE_DEVICES=0 timeout 120 python tools/microbench.py qgz > $O/mb.log 2>&1
CUDA_VISIBLE_DEVICES=0 ZPP_NO_TBL=1 timeout 120 python tools/microbench.py qgz > $O/mb_notbl.log 2>&1
for X in 4 2; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2952$X tools/stage_timeline.py $X > $O/tl4_$X.log 2> $O/tl4_$X.err
  ZPP_QGZ_PULL=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2953$X tools/stage_timeline.py $X > $O/tl4_${X}_pull.log 2> $O/tl4_${X}_pull.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 tools/stage_timeline.py 2 > $O/tl2_2.log 2> $O/tl2_2.err
