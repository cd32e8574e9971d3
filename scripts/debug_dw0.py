import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, numpy as np
from test_gpu_tensorcore import _mlp_io, _fwd, _bwd, _relmax
from paper_1711_06505_b200 import _lib as L0
for prec in ("tf32", "bf16"):
    for U in (1, 64, 300, 3000):
        pdt = "bf16" if prec == "bf16" else "fp32"
        L, pool, rows, p, rt, cnt, cap = _mlp_io(U, 6000, seed=U, dtype=pdt)
        ref = _fwd(L, pool, p, rt, cnt, cap, L0.PREC_FP32)
        got = _fwd(L, pool, p, rt, cnt, cap, L0.PRECISIONS[prec])
        torch.cuda.synchronize()
        demb = torch.randn((cap, 12), device="cuda") * 1e-2
        gr = _bwd(L, pool, p, rt, cnt, cap, L0.PREC_FP32, ref[0], ref[1], demb, ref[3], ref[4])
        gg = _bwd(L, pool, p, rt, cnt, cap, L0.PRECISIONS[prec], ref[0], ref[1], demb, got[3], got[4])
        a, b = gg["w0"].cpu().numpy(), gr["w0"].cpu().numpy()
        nzr = (np.abs(a).sum(1) > 0).mean(); nzc = (np.abs(a).sum(0) > 0).mean()
        print(prec, U, "act0 err", _relmax(got[0][:U], ref[0][:U]), "dw0 err", _relmax(gg["w0"], gr["w0"]),
              "nonzero rows", nzr, "cols", nzc, "ratio", np.abs(a).sum() / max(np.abs(b).sum(), 1e-30), flush=True)
        if U == 300:
            # correlation structure: is it transposed / permuted?
            print("  corr direct", np.corrcoef(a.ravel(), b.ravel())[0, 1], flush=True)
