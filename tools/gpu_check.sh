# Round check on a 4-GPU box (gpurun --gpus 4 -- 'bash tools/gpu_check.sh'):
# the GPU test suite, then the bench line at N = 1, 2, 4 and the reference arm.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_all.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "rc=$?" >> gpurun_out/b1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "rc=$?" >> gpurun_out/b2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > gpurun_out/b4.json 2> gpurun_out/b4.err; echo "rc=$?" >> gpurun_out/b4.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err
