"""kl_adam_step on 40 M parameters (fp32 p, g, m, v + bf16 mirror): time and achieved GB/s (30 B / param)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
n = 40_000_000
p = torch.zeros(n, device="cuda"); g = torch.randn(n, device="cuda") * 1e-3
m = torch.zeros(n, device="cuda"); v = torch.zeros(n, device="cuda")
wc = torch.empty(n, device="cuda", dtype=torch.bfloat16); t = torch.ones(1, dtype=torch.int32, device="cuda")
f = lambda: _capi.call("kl_adam_step", n, 1e-3, 0.9, 0.999, 1e-8, 0, t.data_ptr(), p.data_ptr(), g.data_ptr(),
                       m.data_ptr(), v.data_ptr(), wc.data_ptr(), _capi._stream())
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"adam 40M: {ms*1e3:.1f} us, {30 * n / ms / 1e6:.0f} GB/s")
