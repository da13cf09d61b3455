# 1-GPU pass: GPU tests, config-1 balanced-grid A/B, then the round's profile
# evidence (launch list of bench.py + ncu --set full of each hot kernel).
O=gpurun_out/pr1; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests -q -m gpu -x > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python tools/config1_probe.py > $O/config1_balanced.txt 2>&1
ZPP_BALANCED_GRID=0 timeout 300 python tools/config1_probe.py > $O/config1_unbalanced.txt 2>&1
for c in k1 k2 k3 c1q c1d; do timeout 120 python tools/profile_kernels.py $c 20 >> $O/kernels_r2.jsonl 2>&1; done
TRAFFIC_OUT=$O/ncu_traffic_r2.json bash tools/profile_round.sh r2 > $O/profile_round.log 2>&1
mv gpurun_out/ncu_launches_r2.csv gpurun_out/ncu_full_r2_*.csv gpurun_out/kernels_r2.jsonl gpurun_out/plain_r2.log $O/ 2>/dev/null
du -sh gpurun_out; find gpurun_out -size +8M -print -delete
