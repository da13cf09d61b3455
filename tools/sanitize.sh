# compute-sanitizer evidence for the mbarrier/TMA kernels and the cross-GPU
# barrier protocol.  ONE tool per gpurun call (running several
# tools in one call has left B200 boxes unusable), on a 2-GPU box:
#   gpurun --gpus 2 -- 'TOOL=racecheck OUT=gpurun_out/san bash tools/sanitize.sh'
# Single process: the TMA-fed K2/K3 (ZPP_FORCE_TMA=1), the multi-source TMA
# gather (dequant16_tma_kernel) and the world-1 communicator.  Two ranks:
# tests/dist_worker.py (qwZ, hpZ, qgZ pull and push over CUDA IPC peer memory,
# device barriers) with every rank under the sanitizer.  Each command first
# ran clean without the sanitizer in the round's GPU test pass.
O=${OUT:-gpurun_out/san}; mkdir -p $O
TOOL=${TOOL:-memcheck}
CS="compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20"
ZPP_FORCE_TMA=1 timeout 1200 $CS python -m pytest -q -x -p no:cacheprovider tests/test_gpu_codec.py \
  -k "fused_fixed_fanin or dequant_reduce_many_sources" > $O/${TOOL}_single.log 2>&1
echo "rc=$?" >> $O/${TOOL}_single.log
timeout 900 $CS python -m pytest -q -x -p no:cacheprovider tests/test_gpu_comm_single.py > $O/${TOOL}_comm1.log 2>&1
echo "rc=$?" >> $O/${TOOL}_comm1.log
timeout 900 $CS python -m pytest -q -x -p no:cacheprovider tests/test_gpu_collectives.py -k "qwz_golden" \
  > $O/${TOOL}_gather.log 2>&1
echo "rc=$?" >> $O/${TOOL}_gather.log
export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1
for mode in pull push; do
  export MASTER_PORT=$((29600 + RANDOM % 300)) ZPP_QGZ_MODE=$mode
  pids=()
  for r in 0 1; do
    RANK=$r LOCAL_RANK=$r timeout 1200 $CS python tests/dist_worker.py --group 2 --stages 2 \
      > $O/${TOOL}_dist2_${mode}_rank$r.log 2>&1 &
    pids+=($!)
  done
  for r in 0 1; do wait ${pids[$r]}; echo "rc=$?" >> $O/${TOOL}_dist2_${mode}_rank$r.log; done
done
grep -H "ERROR SUMMARY\|rc=" $O/${TOOL}_*.log > $O/${TOOL}_summary.txt
