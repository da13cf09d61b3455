# 4-GPU check of the hop-2 push: multi-GPU tests, qgZ bucket A/B (hop 2 push
# vs pull) at 2x2 and 2x1, stage timelines, and the 1-GPU span A/B.
O=gpurun_out/hop2; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k "two_gpus or four_gpus or hop1 or large_four" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for NX in "4 2" "2 1"; do
  set -- $NX
  for h in push pull; do
    ZPP_QGZ_HOP2=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $2 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"hop2\": \"$h\"}/" >> $O/qgz.jsonl
  done
done
for h in push pull; do
  ZPP_QGZ_HOP2=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/stage_timeline.py 2 2>>$O/err.log | head -1 | sed "s/}\$/, \"hop2\": \"$h\"}/" >> $O/tl.jsonl
done
export CUDA_VISIBLE_DEVICES=0
for v in 0 1; do ZPP_NO_SPAN=$v timeout 120 python tools/profile_kernels.py qgz1 20 2>>$O/err.log | sed "s/}\$/, \"no_span\": $v}/" >> $O/qgz1.jsonl; done
