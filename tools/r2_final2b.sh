O=${OUT:-gpurun_out/f2b}; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/b1.json 2> $O/b1.err; echo "rc=$?" >> $O/b1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo "rc=$?" >> $O/b2.err
