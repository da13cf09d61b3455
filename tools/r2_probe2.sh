# 2-GPU probe pass: config-1 split, fused N=1 on two input distributions,
# NVLink byte counters, prefetch SM sweep, cross-bucket qgZ sweep at N=2,
# one-rank ncu debug with progress prints.
O=${OUT:-gpurun_out/p2}; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/config1_probe.py > $O/config1.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/microbench.py fused > $O/fused.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/microbench.py qgz > $O/qgz_kernels.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29531 tools/nvl_counters.py 2 > $O/nvl_counters_n2.json 2> $O/nvl_counters.err
for k in default 20 40 59 74; do
  if [ $k = default ]; then timeout 300 $TR --master-port 29532 tools/qwz_layers_probe.py >> $O/prefetch.jsonl 2>> $O/prefetch.err
  else ZPP_QWZ_PREFETCH_SMS=$k timeout 300 $TR --master-port 29532 tools/qwz_layers_probe.py >> $O/prefetch.jsonl 2>> $O/prefetch.err; fi
done
for args in "ZPP_QGZ_XB=0" "ZPP_QGZ_K1_XB_SMS=60" "ZPP_QGZ_K1_XB_SMS=74" "ZPP_QGZ_K1_XB_SMS=88" "ZPP_QGZ_K1_XB_SMS=100"; do
  env $args timeout 300 $TR --master-port 29533 tools/qgz_stream_probe.py 2 8 1 2>> $O/xb.err | tail -1 >> $O/xb.jsonl
done
N=2 X=2 SKIP=8 COUNT=4 OUT=$O PORT=29571 NCU_TIMEOUT=240 bash tools/ncu_rank0.sh
