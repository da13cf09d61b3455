# K2 A/B on one GPU: product tables, split tables, no tables (tools/microbench.py qgz)
O=${OUT:-gpurun_out/k2ab}; mkdir -p $O
python tools/microbench.py qgz > $O/mb_tbl.txt 2>&1
ZPP_TBL_SPLIT=2 python tools/microbench.py qgz > $O/mb_split.txt 2>&1
ZPP_NO_TBL=1 python tools/microbench.py qgz > $O/mb_notbl.txt 2>&1
