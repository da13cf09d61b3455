#!/bin/bash
# Run on the GPU box (via gpurun) on ONE GPU.  Produces the committed profile
# evidence for round $1:
#   gpurun_out/ncu_launches_$1.csv   every kernel launch of `python bench.py` with its device time
#   gpurun_out/ncu_full_$1_<case>.csv   ncu --set full details of each hot kernel at its bench size
#   gpurun_out/ncu_traffic.json      per-launch DRAM bytes of those kernels (the roofline "traffic")
#   gpurun_out/kernels_$1.jsonl      CUDA-event timings of the same kernels without ncu
set -u
R=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
export CUDA_VISIBLE_DEVICES=0
python bench.py --steps 2 --warmup 3 > $OUT/plain_$R.log 2>&1 || { echo "plain bench failed"; exit 1; }
CASES=${CASES:-"qwz1:quantize_reg_kernel gather4:dequant16_tma_kernel k0:quantize_reg_kernel k1:quantize_reg_kernel k2:drq_tbl_kernel k3:dr_fast_kernel c1q:quantize_reg_kernel c1d:dequant8_f32_kernel"}
for CK in $CASES; do
  C=${CK%%:*}
  python tools/profile_kernels.py $C 20 >> $OUT/kernels_$R.jsonl 2>> $OUT/kernels_$R.err || { echo "case $C failed"; exit 1; }
done
# our kernels only (the synthetic-input generation is torch elementwise work)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/ncu_launches_$R.csv \
    -k regex:"quantize_|dequant|drq_|dr_fast|dr_tma|gather_copy|barrier_kernel|wire_|scales_kernel" \
    python bench.py --steps 2 --warmup 3 > $OUT/ncu_launches_$R.log 2>&1
for CK in $CASES; do
  C=${CK%%:*}; K=${CK##*:}
  ncu --set full --clock-control none --import-source on -k regex:"${K}" -s 2 -c 1 -o /tmp/prof_$C \
      python tools/profile_kernels.py $C > $OUT/ncu_full_${R}_$C.log 2>&1
  ncu -i /tmp/prof_$C.ncu-rep --page details --csv > $OUT/ncu_full_${R}_$C.csv 2>/dev/null
  ncu -i /tmp/prof_$C.ncu-rep --page raw --csv > /tmp/raw_$C.csv 2>/dev/null
done
python - <<'PY'
import csv, json, glob, os
out = {}
names = {"qwz1": "quantize_reg_kernel<deq> (fused qwZ self-gather)",
         "gather4": "dequant16_tma_kernel (gather over NVLink)",
         "k0": "quantize_reg_kernel", "k1": "quantize_reg_kernel<swizzle> (qgZ K1)",
         "k2": "drq_tbl_kernel", "k3": "dr_fast_kernel", "c1q": "quantize_reg_kernel<fp32> (config 1)",
         "c1d": "dequant8_f32_kernel (config 1)"}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for f in glob.glob("/tmp/raw_*.csv"):
    c = os.path.basename(f)[4:-4]
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, u, r = rows[0], rows[1], rows[2]
    try:
        i, j = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        out[names.get(c, c)] = float(r[i].replace(",", "")) * scale.get(u[i], 1) + \
            float(r[j].replace(",", "")) * scale.get(u[j], 1)
    except (ValueError, IndexError):
        pass
json.dump(out, open(os.environ.get("TRAFFIC_OUT", "gpurun_out/ncu_traffic.json"), "w"), indent=1)
print(out)
PY
