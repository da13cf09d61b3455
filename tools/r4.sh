mkdir -p gpurun_out
P=29800
run() { # nproc X chunks fused
  P=$((P+1))
  ZPP_QGZ_FUSED=$4 ZPP_QGZ_CHUNKS=$3 ZPP_BENCH_STAGES=1 ZPP_BENCH_SECTIONS=qgz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P tools/bench_zeropp.py $2 2>>gpurun_out/qf.err | grep '^{' | sed "s/^{/{\"chunks\": $3, \"fused\": $4, /" >> gpurun_out/qf.jsonl
}
run 1 1 32 1; run 1 1 32 0
for X in 4 2; do
  for CH in 8 16 32 64; do run 4 $X $CH 1; done
  run 4 $X 32 0
done
