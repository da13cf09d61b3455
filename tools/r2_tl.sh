# 4-GPU: qwZ/qgZ stage timelines at 2x2 and 1x4; GPU-0 A/B of the 1-GPU qgZ
# bucket against the round-start library.
O=gpurun_out/tl; mkdir -p $O
for X in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/stage_timeline.py $X > $O/tl_n4_x$X.jsonl 2>> $O/err.log
done
export CUDA_VISIBLE_DEVICES=0
for r in 1 2; do for L in libzpp_r2start.so libzpp.so; do
  ZPP_LIB=$PWD/paper_2306_10209_b200/$L timeout 120 python tools/profile_kernels.py qgz1 20 2>>$O/err.log \
    | sed "s/}\$/, \"lib\": \"$L\"}/" >> $O/qgz1_ab.jsonl
  ZPP_BALANCED_GRID=0 ZPP_LIB=$PWD/paper_2306_10209_b200/$L timeout 120 python tools/profile_kernels.py qgz1 20 2>>$O/err.log \
    | sed "s/}\$/, \"lib\": \"$L\", \"balanced\": 0}/" >> $O/qgz1_ab.jsonl
done; done
