"""gdpa fwd512 at the c4 shape (B=32, T=4096, d=512, H*n_kv=128): time (+ CTA-0 clock stamps with TRACE=1)."""
import ctypes as C, os, sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F
_capi.lib()
B, T, d, HK, n_kv = 32, 4096, 512, 128, 16
g = torch.Generator(device="cuda").manual_seed(0)
S = (torch.randn(B, T, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
Kt = (torch.randn(B, HK, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
Vt = (torch.randn(B, HK, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
codes = [_capi.ACT_CODES[a] if hasattr(_capi, "ACT_CODES") else 0 for a in ("silu", "relu", "identity", "tanh") * 2]
a = F._gdpa_args(S, Kt, Vt, lens, F._codes(["silu", "relu", "identity", "tanh"] * 2), n_kv, 1.0)
Y = torch.empty_like(S)
a.Y = Y.data_ptr()
f = lambda: _capi.call("kl_gdpa_fwd", C.byref(a), _capi._stream())
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): f()
e1.record(); torch.cuda.synchronize()
print(f"gdpa fwd512: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
if os.environ.get("TRACE"):
    tr = torch.zeros(32 * 16, dtype=torch.int64).pin_memory()
    a.trace = tr.data_ptr()
    f(); torch.cuda.synchronize()
    t = tr.view(32, 16); t0 = int(t[0, 0])
    names = ["p_v0", "p_z", "p_zend", "p_v1end", "m_zgo", "m_zend", "m_afull", "m_y0", "m_y1", "e_zfull", "e_a", "e_y0f", "e_y0d", "e_y1f", "e_y1d"]
    for k in range(8):
        print(f"tile {k} " + " ".join(f"{nm}={int(t[k, e]) - t0:7d}" for e, nm in enumerate(names)))
