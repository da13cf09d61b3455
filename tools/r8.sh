mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
python tools/profile_kernels.py k1 5 > gpurun_out/k1_plain.json || exit 1
ncu --set full --import-source on --clock-control none -k regex:quantize_reg_kernel -s 2 -c 1 -o /tmp/k1 python tools/profile_kernels.py k1 > gpurun_out/k1_ncu.log 2>&1
ncu -i /tmp/k1.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_sass.csv 2>gpurun_out/k1_sass.err
ls -la gpurun_out
