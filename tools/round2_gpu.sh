# Round-2 GPU pass on a 4-GPU box: bench lines at N = 1, 2, 4, the reference
# arm, and one-rank ncu captures under real peer traffic (1x4 and 2x2).
O=${OUT:-gpurun_out/r2}; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/b1.json 2> $O/b1.err; echo "rc=$?" >> $O/b1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo "rc=$?" >> $O/b2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo "rc=$?" >> $O/b4.err
N=4 X=4 SKIP=8 COUNT=4 OUT=$O PORT=29571 bash tools/ncu_rank0.sh
N=4 X=2 SKIP=10 COUNT=5 OUT=$O PORT=29572 bash tools/ncu_rank0.sh
