#!/bin/bash
# Run on the GPU box (via gpurun) after `python bench.py` has exited 0 there.
# Produces the committed profile evidence for round $1:
#   gpurun_out/ncu_launches_$1.csv   every kernel launch of the bench command with its device time
#   gpurun_out/ncu_full_$1_*.csv     ncu --set full details of the dominant kernels
#   gpurun_out/ncu_traffic.json      per-launch DRAM bytes of those kernels (roofline "traffic")
set -u
R=${1:-r1}
OUT=gpurun_out
python bench.py --steps 2 --warmup 3 > $OUT/plain_$R.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/ncu_launches_$R.csv \
    python bench.py --steps 2 --warmup 3 > $OUT/ncu_launches_$R.log 2>&1
for K in quantize_reg_kernel dequant_reduce16_kernel drq16_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"${K}" -s 2 -c 1 -o /tmp/prof_$K \
      python bench.py --steps 2 --warmup 3 > $OUT/ncu_full_${R}_$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page details --csv > $OUT/ncu_full_${R}_$K.csv 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > /tmp/raw_$K.csv 2>/dev/null
done
python - <<'EOF'
import csv, json, glob, os
out = {}
names = {"quantize_reg_kernel": "quantize_reg_kernel<deq> (fused qwZ self-gather)",
         "drq16_kernel": "drq16_kernel", "dequant_reduce16_kernel": "dequant_reduce16_kernel"}
for f in glob.glob("/tmp/raw_*.csv"):
    k = os.path.basename(f)[4:-4]
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, r = rows[0], rows[2]
    def g(name):
        try:
            return float(r[h.index(name)].replace(",", ""))
        except Exception:
            return None
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    ur, uw = rows[1][h.index("dram__bytes_read.sum")], rows[1][h.index("dram__bytes_write.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd is not None and wr is not None:
        out[names.get(k, k)] = rd * scale.get(ur, 1) + wr * scale.get(uw, 1)
json.dump(out, open("gpurun_out/ncu_traffic.json", "w"), indent=1)
print(out)
EOF
