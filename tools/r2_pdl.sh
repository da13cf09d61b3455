# 4-GPU: tests with PDL on, then PDL A/B on qgZ buckets (2x2, 1x4, 2x1) and
# the 40-layer qwZ forward.
O=gpurun_out/pdl; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in 1 0; do
  for NX in "4 2" "4 4" "2 1"; do
    set -- $NX
    ZPP_PDL=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $2 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"pdl\": $v}/" >> $O/qgz.jsonl
  done
  ZPP_PDL=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qwz_layers_probe.py 2>>$O/err.log | tail -1 | sed "s/}\$/, \"pdl\": $v}/" >> $O/qwz.jsonl
done
