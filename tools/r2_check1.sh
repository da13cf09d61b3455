# One-GPU pass: single-GPU tests, smoke, bench N=1 and the reference arm.
O=${OUT:-gpurun_out/c1}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --ignore=tests/test_gpu_dist.py > $O/t1.log 2>&1; echo "tests rc=$?" >> $O/t1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/b1.json 2> $O/b1.err; echo "rc=$?" >> $O/b1.err
timeout 300 python bench.py --impl reference > $O/bref.json 2> $O/bref.err; echo "rc=$?" >> $O/bref.err
