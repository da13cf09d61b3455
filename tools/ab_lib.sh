# A/B of builds of libzpp on one GPU: $1 = profile_kernels cases, $2.. = library
# file names in paper_2306_10209_b200/ (build the variants first, e.g. every
# csrc/*.cu with nvcc ... -DZPP_PIPE_DEQ=1 -c, then nvcc -shared -o libzpp_alt.so *.o -lcuda)
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
CASES=$1; shift
for r in 1 2; do for L in "$@"; do for C in $CASES; do
  echo -n "$L " >> gpurun_out/ab.log
  ZPP_LIB=$PWD/paper_2306_10209_b200/$L python tools/profile_kernels.py $C 20 >> gpurun_out/ab.log 2>&1
done; done; done
