# qgZ stage/SM-split sweep on the GPUs of one box: bash tools/qgz_sweep.sh N X
N=${1:-4}; X=${2:-4}
mkdir -p gpurun_out
for K in 0 24 36 48 64; do
  if [ $K = 0 ]; then unset ZPP_QGZ_K1_SMS; else export ZPP_QGZ_K1_SMS=$K; fi
  ZPP_BENCH_SECTIONS=qgz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29600 + K)) tools/bench_zeropp.py $X 2>>gpurun_out/qgz_sweep.err
done
