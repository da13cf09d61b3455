import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp
lib = zpp._lib.load()
st = torch.cuda.current_stream().cuda_stream
bits = torch.arange(0, 1 << 27, dtype=torch.int64, device="cuda").to(torch.int32)
m = bits.view(torch.float32)
out = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
zpp._lib.check(lib.zpp_scales(m.data_ptr(), zpp._lib.F32, 1 << 27, 8, out.data_ptr(), st))
md = m.double()
want = md / 127.0
bad = (out != want).nonzero().flatten()
print("mismatches", bad.numel())
for i in bad[:10].tolist():
    print(i, hex(i), m[i].item(), md[i].item(), out[i].item(), want[i].item())
# compare conversions: torch's float->double vs exact
print("md zero count for nonzero bits:", int(((md == 0) & (bits != 0)).sum()))
