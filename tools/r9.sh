mkdir -p gpurun_out
P=29900
for N in 4 2; do
for PC in 1 2 3 4; do for KS in 24 37 56; do
  if [ $PC = 1 ] && [ $KS != 37 ]; then continue; fi
  P=$((P+1))
  ZPP_QWZ_PIECES=$PC ZPP_QWZ_K0_SMS=$KS timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P tools/bench_gather.py 2>/dev/null | grep '^{' | sed "s/^{/{\"pieces\": $PC, \"k0_sms\": $KS, /" >> gpurun_out/qp.jsonl
done; done; done
