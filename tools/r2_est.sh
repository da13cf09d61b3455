# K2 certified-estimate kernel: GPU tests (single + 2/4-GPU), kernel A/B
# (ZPP_K2=tbl vs default), qgZ bucket A/B at 2x2 and 2x1.
O=gpurun_out/est; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
export CUDA_VISIBLE_DEVICES=0
for r in 1 2; do for v in est tbl; do for c in k2 qgz1; do
  ZPP_K2=$v timeout 120 python tools/profile_kernels.py $c 20 2>>$O/err.log | sed "s/}\$/, \"k2\": \"$v\"}/" >> $O/kernels.jsonl
done; done; done
ZPP_K2=est timeout 120 python tools/microbench.py qgz > $O/mb_est.txt 2>&1
ZPP_K2=tbl timeout 120 python tools/microbench.py qgz > $O/mb_tbl.txt 2>&1
unset CUDA_VISIBLE_DEVICES
for v in est tbl; do for NX in "4 2" "2 1"; do
  set -- $NX
  ZPP_K2=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $2 8 1 2>>$O/err.log | tail -1 | sed "s/}\$/, \"k2\": \"$v\"}/" >> $O/qgz.jsonl
done; done
