# Same-box A/B of the round-start library (libzpp_r2start.so, built from
# 709e830's csrc) against the current one, per kernel case, two rounds.
O=${OUT:-gpurun_out/ab}; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
for r in 1 2; do
  for c in qwz1 k0 gather4 k1 k2 k3 c1q c1d; do
    for L in libzpp_r2start.so libzpp.so; do
      ZPP_LIB=$PWD/paper_2306_10209_b200/$L timeout 120 python tools/profile_kernels.py $c 20 2>>$O/err.log \
        | sed "s/}\$/, \"lib\": \"$L\", \"round\": $r}/" >> $O/ab.jsonl
    done
  done
done
