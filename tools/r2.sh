mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "b2 rc=$?" >> gpurun_out/b2.err
bash tools/qgz_sweep.sh 4 4 > gpurun_out/qs44.jsonl
bash tools/qgz_sweep.sh 4 2 > gpurun_out/qs42.jsonl
