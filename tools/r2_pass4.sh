# 4-GPU pass: cross-bucket qgZ sweep (1x4, 2x2, and 1x2 on two GPUs), qwZ
# prefetch sweeps at N = 4 and 2, the fused N = 1 pass after a 1 s warm-up, bench at N = 4, then one
# ncu capture of rank 0 under peer traffic (2x2).
O=${OUT:-gpurun_out/p4}; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "four_gpus or qgz_hop1 or two_gpus" > $O/t4.log 2>&1; echo "tests rc=$?" >> $O/t4.log
nvidia-smi nvlink -gt d -i 0 > $O/nvlink_gt_probe.txt 2>&1
CUDA_VISIBLE_DEVICES=0 ZPP_MB_WARM_S=1.0 timeout 300 python tools/microbench.py fused > $O/fused_longwarm.txt 2>&1
pf() {  # env...
  env "$@" timeout 300 $TR --master-port $((29543 + RANDOM % 100)) tools/qwz_layers_probe.py 2>> $O/prefetch.err \
    | tail -1 | sed "s/}\$/, \"env\": \"$*\"}/" >> $O/prefetch.jsonl
}
pf ZPP_QWZ_GATHER_OCC=2
pf ZPP_QWZ_GATHER_OCC=1
pf ZPP_QWZ_GATHER_OCC=3
pf ZPP_QWZ_PREFETCH_MODE=split ZPP_QWZ_PREFETCH_SMS=20
pf ZPP_QWZ_PREFETCH_MODE=split ZPP_QWZ_PREFETCH_SMS=30
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
pf ZPP_QWZ_GATHER_OCC=2
pf ZPP_QWZ_GATHER_OCC=1
pf ZPP_QWZ_PREFETCH_MODE=split ZPP_QWZ_PREFETCH_SMS=40
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
OUT=$O bash tools/qgz_xb_sweep.sh
timeout 900 $TR --master-port 29544 bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo "rc=$?" >> $O/b4.err
N=4 X=2 SKIP=10 COUNT=5 OUT=$O PORT=29571 NCU_TIMEOUT=420 bash tools/ncu_rank0.sh
du -sh $O; find $O -size +8M -print -delete
