# Round check on a 4-GPU box (gpurun --gpus 4 -- 'OUT=gpurun_out/x bash tools/gpu_check.sh'):
# the GPU test suite, then the bench line at N = 1, 2, 4 and the reference arm.
O=${OUT:-gpurun_out}
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/t_all.log 2>&1; echo "tests rc=$?" >> $O/t_all.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > $O/b1.json 2> $O/b1.err; echo "rc=$?" >> $O/b1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo "rc=$?" >> $O/b2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo "rc=$?" >> $O/b4.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > $O/bref.json 2> $O/bref.err
