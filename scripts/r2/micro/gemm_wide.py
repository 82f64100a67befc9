"""Weight-gradient GEMM shapes (fp32 accumulate) through the wide CTA-pair path vs KL_GEMM_NOWIDE: error + time."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
def t(fn, n=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
torch.manual_seed(0)
for (M, N, Kb, nb) in ((1536, 512, 4096, 32), (512, 512, 4096, 32), (768, 256, 1024, 128), (256, 256, 1024, 128), (1024, 1024, 4096, 8), (768, 512, 1000, 7)):
    K = Kb * nb
    A3 = torch.randn(nb, Kb, M, device="cuda").bfloat16()   # dY rows -> A = dY^T (MN-major), batch-reduced
    B3 = torch.randn(nb, Kb, N, device="cuda").bfloat16()
    ref = torch.einsum("bkm,bkn->mn", A3.float(), B3.float())
    for kmaj in (False, True):
        if kmaj:
            A = A3.transpose(1, 2).contiguous(); Bm = B3.transpose(1, 2).contiguous()
            fa, fb = A, Bm.transpose(1, 2)
        else:
            fa, fb = A3.transpose(1, 2), B3
        C = torch.zeros(M, N, device="cuda")
        _capi.gemm(fa, fb, C, beta=1.0, reduce=(False, True))
        err = ((C - ref).norm() / ref.norm()).item()
        ms = t(lambda: _capi.gemm(fa, fb, C, beta=1.0, reduce=(False, True)))
        print(f"{M}x{N}x{K} {'Kmaj' if kmaj else 'MNmaj'} {os.environ.get('KL_GEMM_NOWIDE') and 'nowide' or 'wide'}: "
              f"{ms*1e3:7.1f} us {2*M*N*K/ms/1e9:6.0f} TF/s  err {err:.2e}", flush=True)
