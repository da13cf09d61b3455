O=gpurun_out/x1; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k "two_gpus or hop1" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in 1 0; do
  ZPP_QGZ_X1=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py 1 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"x1\": $v}/" >> $O/qgz.jsonl
done
