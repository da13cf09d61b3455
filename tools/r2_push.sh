O=gpurun_out/push; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x -k "two_gpus or four_gpus or hop1 or large_four" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for v in 0 1; do for NX in "4 2" "2 1"; do
  set -- $NX
  ZPP_PUSH_STAGE_SELF=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $2 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"stage_self\": $v}/" >> $O/qgz.jsonl
done; done
