# Cross-bucket qgZ overlap sweep (K1 of bucket b+1 beside K2/K3 of bucket b):
# off; SM split with K1 budgets; SM sharing (both grids on every SM).
#   gpurun --gpus 4 -- 'OUT=gpurun_out/xb bash tools/qgz_xb_sweep.sh'
O=${OUT:-gpurun_out/xb}; mkdir -p $O
run() {  # N X NB S env...
  local N=$1 X=$2 NB=$3 S=$4; shift 4
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/qgz_stream_probe.py $X $NB $S 2>>$O/err.log | tail -1 \
    | sed "s/}\$/, \"env\": \"$*\"}/" >> $O/sweep.jsonl
}
for NX in "4 4" "4 2" "2 2"; do
  set -- $NX
  run $1 $2 8 1 ZPP_QGZ_XB=0
  for k in 60 74; do run $1 $2 8 1 ZPP_QGZ_XB=1 ZPP_QGZ_K1_XB_SMS=$k; done
  for o in 1 2; do run $1 $2 8 1 ZPP_QGZ_XB=1 ZPP_QGZ_XB_MODE=share ZPP_QGZ_K2_OCC=$o; done
done
# one bucket in two stages (extra barriers), K1 share swept
for NX in "4 4" "4 2"; do
  set -- $NX
  run $1 $2 1 1 ZPP_QGZ_XB=1
  for k in 49 74; do run $1 $2 1 2 ZPP_QGZ_K1_SMS=$k; done
done
