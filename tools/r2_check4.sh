# Four-GPU pass: multi-GPU tests, bench lines at N = 2 and 4, one-rank ncu captures under peer traffic.
O=${OUT:-gpurun_out/c4}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py -v -m gpu > $O/t4.log 2>&1; echo "tests rc=$?" >> $O/t4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo "rc=$?" >> $O/b2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo "rc=$?" >> $O/b4.err
N=4 X=4 SKIP=8 COUNT=4 OUT=$O PORT=29571 bash tools/ncu_rank0.sh
N=4 X=2 SKIP=10 COUNT=5 OUT=$O PORT=29572 bash tools/ncu_rank0.sh
