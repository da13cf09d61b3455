mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for i in 1 2 3; do for MB in 2 3 4; do ZPP_QDEQ_MINB=$MB python tools/profile_kernels.py qwz1 50 | sed "s/^{/{\"minb\": $MB, /" >> gpurun_out/k.jsonl; done; done
