# compute-sanitizer evidence for the mbarrier/TMA kernels and the cross-GPU
# barrier protocol.  Run on a >= 2-GPU box:
#   gpurun --gpus 2 -- 'OUT=gpurun_out/san bash tools/sanitize.sh'
# Single process: the TMA-fed K2/K3 (ZPP_FORCE_TMA=1), the multi-source TMA
# gather (dequant16_tma_kernel) and the world-1 communicator, under memcheck,
# racecheck (shared-memory hazards) and synccheck (barrier / mbarrier misuse).
# Two ranks: tests/dist_worker.py (qwZ, hpZ, qgZ push and pull over CUDA IPC
# peer memory, device barriers) with every rank under the sanitizer.
O=${OUT:-gpurun_out/san}; mkdir -p $O
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
K="fused_fixed_fanin or dequant_reduce_many_sources or gather"
for tool in memcheck racecheck synccheck; do
  ZPP_FORCE_TMA=1 timeout 1500 $CS --tool $tool python -m pytest -q -x -p no:cacheprovider tests/test_gpu_codec.py \
    -k "$K" > $O/single_$tool.log 2>&1; echo "rc=$?" >> $O/single_$tool.log
  timeout 900 $CS --tool $tool python -m pytest -q -x -p no:cacheprovider tests/test_gpu_comm_single.py \
    > $O/comm1_$tool.log 2>&1; echo "rc=$?" >> $O/comm1_$tool.log
done
for tool in memcheck racecheck synccheck; do
  for mode in push pull; do
    export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$((29600 + RANDOM % 300)) ZPP_QGZ_MODE=$mode
    pids=()
    for r in 0 1; do
      RANK=$r LOCAL_RANK=$r timeout 1500 $CS --tool $tool python tests/dist_worker.py --group 2 --stages 2 \
        > $O/dist2_${mode}_${tool}_rank$r.log 2>&1 &
      pids+=($!)
    done
    for r in 0 1; do wait ${pids[$r]}; echo "rc=$?" >> $O/dist2_${mode}_${tool}_rank$r.log; done
  done
done
grep -H "ERROR SUMMARY\|rc=" $O/*.log > $O/summary.txt
