# One-rank ncu capture of the fused collectives under real NVLink peer traffic:
# ranks 1..N-1 run plainly, rank 0 under ncu (--set full plus NVLink rx/tx
# bytes), kernels filtered to the data plane (gather, K1 push, K2, K3).
#   N=4 X=4 OUT=gpurun_out/x bash tools/ncu_rank0.sh
# The GPU box's ncu first runs the profiled command once without ncu, then
# again under ncu, so the peers run the workload twice, back to back (each
# run is a fresh rendezvous on the same port).
N=${N:-4}; X=${X:-$N}; O=${OUT:-gpurun_out}; PORT=${PORT:-29561}
# warm-up launches matching the filter: 4 per iteration with one group (K0, gather, K1, K2), 5 with two (K0, gather, K1-push, K2, K3): SKIP=8 COUNT=4 or SKIP=10 COUNT=5
mkdir -p $O
export WORLD_SIZE=$N MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT
T=${NCU_TIMEOUT:-600}
for r in $(seq 1 $((N - 1))); do
  (for pass in plain ncu; do
     RANK=$r LOCAL_RANK=$r timeout $T python tools/nvl_profile.py $X >> $O/nvl_rank$r.log 2>&1
     echo "rank $r $pass pass rc=$?" >> $O/nvl_rank$r.log
   done) &
done
RANK=0 LOCAL_RANK=0 timeout $T ncu --set full --clock-control none --import-source on \
  --metrics nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"dequant16_tma_kernel|drq_tma_kernel|dr_tma_kernel|quantize_push_kernel|drq_tbl_kernel|quantize_reg_kernel" \
  --launch-skip ${SKIP:-8} --launch-count ${COUNT:-4} -o /tmp/nvl_n${N}_x${X} -f python tools/nvl_profile.py $X > $O/nvl_rank0.log 2>&1
echo "rank0 rc=$?" >> $O/nvl_rank0.log
wait
# the report stays on the box (gpurun copies back at most 64 MiB): CSV pages only
if [ -f /tmp/nvl_n${N}_x${X}.ncu-rep ]; then
  ncu -i /tmp/nvl_n${N}_x${X}.ncu-rep --page raw --csv > $O/nvl_n${N}_x${X}_raw.csv 2>&1
  ncu -i /tmp/nvl_n${N}_x${X}.ncu-rep --page details --csv > $O/nvl_n${N}_x${X}_details.csv 2>&1
fi
