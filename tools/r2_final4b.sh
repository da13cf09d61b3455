# Round-2 final confirmation on a 4-GPU box: GPU suite, smoke, bench lines at
# N = 1, 2, 4, the reference arm, and a one-rank NVLink ncu capture at N = 2.
O=${OUT:-gpurun_out/f4b}; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/b1.json 2> $O/b1.err; echo "rc=$?" >> $O/b1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo "rc=$?" >> $O/b2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo "rc=$?" >> $O/b4.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > $O/bref.json 2> $O/bref.err; echo "rc=$?" >> $O/bref.err
N=2 X=2 SKIP=8 COUNT=4 OUT=$O PORT=29573 NCU_TIMEOUT=420 bash tools/ncu_rank0.sh
du -sh gpurun_out; find gpurun_out -size +8M -print -delete
