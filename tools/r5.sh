mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t_dist.log 2>&1; echo "rc=$?" >> gpurun_out/t_dist.log
P=29800
run() { # nproc X chunks pfrac tag trace
  P=$((P+1))
  if [ "$6" = 1 ]; then export ZPP_QGZ_TRACE=gpurun_out/tr_$5; else unset ZPP_QGZ_TRACE; fi
  ZPP_QGZ_PFRAC=$4 ZPP_QGZ_CHUNKS=$3 ZPP_BENCH_STAGES=1 ZPP_BENCH_SECTIONS=qgz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P tools/bench_zeropp.py $2 2>>gpurun_out/qf.err | grep '^{' | sed "s/^{/{\"tag\": \"$5\", \"trace\": $6, /" >> gpurun_out/qf.jsonl
}
run 1 1 32 0.5 w1 1
run 4 4 32 0.5 x4 1
run 4 2 32 0.5 x2 1
run 1 1 32 0.5 w1 0
for CH in 16 32; do for PF in 0.4 0.5 0.6; do run 4 4 $CH $PF x4c${CH}p$PF 0; run 4 2 $CH $PF x2c${CH}p$PF 0; done; done
python tools/qgz_trace_summary.py gpurun_out/tr_*_rank0.bin > gpurun_out/trace_summary.txt 2>&1
rm -f gpurun_out/tr_*rank[123].bin
