# 2-GPU check of the warp-coalesced fp32 span layout (K3, K2 final output):
# GPU tests, then A/B (ZPP_NO_SPAN=1) of the kernels and of qgZ buckets.
O=gpurun_out/span; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in 0 1; do
  for c in k3 k2; do ZPP_NO_SPAN=$v CUDA_VISIBLE_DEVICES=0 timeout 120 python tools/profile_kernels.py $c 20 | sed "s/}\$/, \"no_span\": $v}/" >> $O/kernels.jsonl 2>&1; done
  for X in 1 2; do
    ZPP_NO_SPAN=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $X 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"no_span\": $v}/" >> $O/qgz.jsonl
  done
done
