# Late bucket pipelining (K1 of bucket b+1 beside K3 of bucket b) with a second hop.
O=gpurun_out/late; mkdir -p $O
run() {  # N X env...
  local N=$1 X=$2; shift 2
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $X 8 1 2>>$O/err.log | tail -1 \
    | sed "s/}\$/, \"env\": \"$*\"}/" >> $O/sweep.jsonl
}
for NX in "4 2" "2 1"; do
  set -- $NX
  run $1 $2 ZPP_QGZ_XB=0
  for k in 60 74 100 120; do run $1 $2 ZPP_QGZ_XB_LATE=1 ZPP_QGZ_K1_XB_SMS=$k; done
done
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "two_gpus_bucket" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
