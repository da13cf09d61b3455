# Same-box A/B of the round-start library (libzpp_r2start.so, built from
# 709e830's csrc) against the current one, per kernel case, two rounds.
O=${OUT:-gpurun_out/ab}; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
for r in 1 2; do
  for c in qwz1 k0 gather4 k1 k2 k3 c1q c1d; do
    for L in libzpp_r2start.so libzpp.so; do
      ZPP_LIB=$PWD/paper_2306_10209_b200/$L timeout 120 python tools/profile_kernels.py $c 20 2>>$O/err.log \
        | sed "s/}\$/, \"lib\": \"$L\", \"round\": $r}/" >> $O/ab.jsonl
    done
  done
done
# qgZ at N = 1 (1x1): span layout and bucket pipelining A/B
for v in 0 1; do for xb in 0 2; do
  ZPP_NO_SPAN=$v ZPP_QGZ_XB=$xb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py 1 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"no_span\": $v}/" >> $O/qgz_n1.jsonl
done; done
TRAFFIC_OUT=$O/ncu_traffic_r2b.json bash tools/profile_round.sh r2b > $O/profile_round.log 2>&1
mv gpurun_out/ncu_launches_r2b.csv gpurun_out/ncu_full_r2b_*.csv gpurun_out/kernels_r2b.jsonl $O/ 2>/dev/null
rm -f gpurun_out/*.log
du -sh gpurun_out; find gpurun_out -size +8M -print -delete
