"""Micro-benchmark of the tcgen05 swap-AB GEMM alone (is_dbg_gemm), with optional
per-CTA globaltimer stamps (IS_GEMM_STAMPS=<device ptr>)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2506_22950_b200 import _lib

torch.cuda.set_device(0)
shapes = [(2048, 2048, 16, 8), (2048, 2048, 16, 4), (2048, 2048, 16, 2), (4096, 2048, 16, 4), (12288, 2048, 16, 1),
          (12288, 2048, 16, 2), (12288, 2048, 16, 3), (2048, 6144, 16, 8), (151936, 2048, 16, 1)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M, K, R, S in shapes:
    w = (torch.randn(M, K, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(R, K, device="cuda").to(torch.bfloat16)
    y = torch.zeros(R, M, device="cuda")
    for _ in range(3):
        _lib.is_dbg_gemm(w, x, y, split=S)
    ts = []
    for cold in (0, 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tt = []
        for _ in range(20):
            if cold:
                flush.zero_()
            e0.record()
            _lib.is_dbg_gemm(w, x, y, split=S)
            e1.record()
            torch.cuda.synchronize()
            tt.append(e0.elapsed_time(e1))
        ts.append(np.median(tt) * 1e3)
    mb = M * K * 2 / 1e6
    print(f"M={M:6d} K={K} R={R} split={S}: warm {ts[0]:7.2f} us  cold {ts[1]:7.2f} us  ({mb:.1f} MB -> {mb / ts[1] * 1e3 / 1e3:.2f} TB/s cold)")
    # stamps
    n_cta = ((M + 127) // 128) * S if S > 1 else min((M + 127) // 128, 148)
    st = torch.zeros(n_cta * 16, dtype=torch.int64, device="cuda")
    os.environ["IS_GEMM_STAMPS"] = str(st.data_ptr())
    flush.zero_()
    torch.cuda.synchronize()
    _lib.is_dbg_gemm(w, x, y, split=S)
    torch.cuda.synchronize()
    del os.environ["IS_GEMM_STAMPS"]
    a = st.view(n_cta, 16).cpu().numpy().astype(np.float64)
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    names = ["start", "setup", "tma0", "full0", "fullN", "tfull", "red_w", "cbar1", "reduce", "epi", "cbar2", "end"]
    med = np.median(rel[:, :12], axis=0)
    mx = np.max(rel[:, :12], axis=0)
    print("   median us: " + " ".join(f"{n}={v:.2f}" for n, v in zip(names, med)))
    print("   max    us: " + " ".join(f"{n}={v:.2f}" for n, v in zip(names, mx)))
