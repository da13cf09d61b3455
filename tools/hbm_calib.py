"""HBM calibration: write-only, read-only and copy bandwidth with torch ops."""
import torch
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s=torch.cuda.Event(True); e=torch.cuda.Event(True); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/it*1e-3
n = 1 << 30
a = torch.empty(n, dtype=torch.float16, device="cuda"); b = torch.empty(n, dtype=torch.float16, device="cuda")
a.normal_()
s = t(lambda: b.fill_(1.0)); print(f"fill (write only) {2*n/s/1e9:.0f} GB/s")
s = t(lambda: b.copy_(a)); print(f"copy              {4*n/s/1e9:.0f} GB/s")
c = torch.empty(n // 2, dtype=torch.int8, device="cuda")
s = t(lambda: torch.sum(a, dtype=torch.float32)); print(f"sum (read only)   {2*n/s/1e9:.0f} GB/s")
d = torch.empty(n // 2, dtype=torch.float16, device="cuda")
x8 = torch.randint(-100, 100, (n // 2,), dtype=torch.int8, device="cuda")
s = t(lambda: d.copy_(x8)); print(f"int8->fp16 cast (1R:2W) {3*(n//2)/s/1e9:.0f} GB/s")
s = t(lambda: c.copy_(d)); print(f"fp16->int8 cast (2R:1W) {3*(n//2)/s/1e9:.0f} GB/s")
import ctypes, glob, os
libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(libs[0])
rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
st = torch.cuda.current_stream().cuda_stream
s = t(lambda: rt.cudaMemsetAsync(b.data_ptr(), 0, 2 * n, st)); print(f"cudaMemset (write only) {2*n/s/1e9:.0f} GB/s")
