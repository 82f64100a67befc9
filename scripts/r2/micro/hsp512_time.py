"""hsp_fwd512 at the c4 shape (B=32, T=4096, d=512, HQ=320): time + parity vs torch fp32."""
import ctypes as C, os, sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
B, T, d, HQ, n1 = 32, 4096, 512, 320, 256
g = torch.Generator(device="cuda").manual_seed(0)
S = (torch.randn(B, T, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
Q = (torch.randn(HQ, d, device="cuda", generator=g) * 2.0).to(torch.bfloat16)
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
if os.environ.get("JAG"):
    lens = torch.randint(0, T + 1, (B,), device="cuda", generator=g).to(torch.int32); lens[1] = 0; lens[2] = 1
O1 = torch.zeros(B, n1, d, device="cuda", dtype=torch.bfloat16)
O2 = torch.zeros(B, HQ - n1, d, device="cuda", dtype=torch.bfloat16)
LSE = torch.zeros(B, HQ, device="cuda")
a = _capi.HspArgs()
a.B, a.T, a.HQ, a.d, a.n1, a.dtype = B, T, HQ, d, n1, _capi.KL_BF16
a.lengths = lens.data_ptr()
a.S, a.s_rs, a.s_bs = S.data_ptr(), S.stride(1), S.stride(0)
a.Q = Q.data_ptr()
a.O1, a.o1_bs, a.O2, a.o2_bs = O1.data_ptr(), O1.stride(0), O2.data_ptr(), O2.stride(0)
a.LSE = LSE.data_ptr()
if not os.environ.get("OLD"):
    nb = int(_capi.lib().kl_hsp_fwd_workspace_bytes(C.byref(a)))
    ws = torch.empty(nb, device="cuda", dtype=torch.uint8)
    a.workspace, a.workspace_bytes = ws.data_ptr(), nb
f = lambda: _capi.call("kl_hsp_fwd", C.byref(a), _capi._stream())
n = int(os.environ.get("N", "20"))
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"hsp_fwd512 B={B} T={T}: {ms*1e3:.1f} us, {4*B*T*HQ*d/ms/1e9:.0f} TF/s algorithmic", flush=True)
if n > 1:
    err = 0.0; lerr = 0.0
    for b in range(B):
        L = int(lens[b])
        if L == 0:
            assert (O1[b] == 0).all() and (O2[b] == 0).all() and torch.isinf(LSE[b]).all(); continue
        Z = Q.float() @ S[b, :L].float().t()
        lse = torch.logsumexp(Z, -1)
        O = torch.softmax(Z, -1) @ S[b, :L].float()
        out = torch.cat([O1[b].float(), O2[b].float()], 0)
        err = max(err, ((out - O).abs().max() / O.abs().max()).item()); lerr = max(lerr, (LSE[b] - lse).abs().max().item())
    print(f"parity: pooled max rel err {err:.3e}, lse abs err {lerr:.3e}")
if os.environ.get("TRACE"):
    tr = torch.zeros(12 * 64, dtype=torch.int64).pin_memory()
    os.environ["KL_HSP_TRACE"] = str(tr.data_ptr())
    f(); torch.cuda.synchronize()
    t = tr.view(12, 64); t0 = int(t[0, 0])
    names = ["p_blk", "p_a0", "p_end", "z_go", "z_a0", "z_end", "o_pw", "o_rw", "s_z", "s_pe", "s_pw", "s_done"]
    for n in range(12):
        print(f"blk {n:2d} " + " ".join(f"{nm}={int(t[e, n]) - t0:7d}" for e, nm in enumerate(names)))
