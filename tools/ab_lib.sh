# Build the B side first, e.g. with a -D switch: for f in paper_2306_10209_b200/csrc/*.cu; do nvcc ... -DZPP_DEQ_FAST_LOOP=0 -c $f; done; nvcc -shared -o paper_2306_10209_b200/libzpp_alt.so *.o -lcuda
# A/B of two builds of libzpp on one GPU: $1 = profile_kernels cases
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
for r in 1 2; do for L in libzpp.so libzpp_alt.so; do for C in $1; do
  echo -n "$L " >> gpurun_out/ab.log
  ZPP_LIB=$PWD/paper_2306_10209_b200/$L python tools/profile_kernels.py $C 20 >> gpurun_out/ab.log 2>&1
done; done; done
