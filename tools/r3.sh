mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t_dist.log 2>&1; echo "rc=$?" >> gpurun_out/t_dist.log
for X in 4 2; do
  ZPP_BENCH_SECTIONS=qgz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2970$X tools/bench_zeropp.py $X >> gpurun_out/qf.jsonl 2>>gpurun_out/qf.err
  ZPP_QGZ_FUSED=0 ZPP_BENCH_SECTIONS=qgz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$X tools/bench_zeropp.py $X >> gpurun_out/qf.jsonl 2>>gpurun_out/qf.err
done
