# qgZ stage timelines at 1x4 and 2x2 for several TMA ring stage sizes (K2/K3)
mkdir -p gpurun_out; rm -f gpurun_out/tts.log
for B in 6144 12288 24576 49152; do for X in 4 2; do
  echo "== bytes=$B X=$X" >> gpurun_out/tts.log
  ZPP_TMA_STAGE_BYTES=$B timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 297$X$((B/6144)) tools/stage_timeline.py $X 2>/dev/null | grep '"rank": 0' >> gpurun_out/tts.log
done; done
