"""DGEMM efficiency probes (one GPU, seconds):
 1. FP64 tensor-pipe ceiling vs warps per SM sub-partition (register-resident
    DMMA chains, hplk_dmma_peak with blocks_per_sm x warps);
 2. the trailing DGEMM at the same m x n for k = 512 and 2048 (a CTA tile's
    mainloop grows with k, its prologue/epilogue do not) under the tile
    configs (gemm_cfg 0/1/2; round 1's epilogue / persistence variants were
    removed after measuring them, profiles/r01_gemm_*).

    python tools/gemm_overhead.py [m] [cfg ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_10397_b200 as H  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cfgs = [int(c) for c in sys.argv[2:]] or [2, 0, 1]
peak = H.hplk_dmma_peak()
for bps, w in ((1, 4), (1, 8), (1, 12), (3, 4), (1, 16), (2, 8), (4, 4)):
    tf = H.hplk_dmma_peak(20000, bps, w)
    print(json.dumps(dict(dmma_blocks_per_sm=bps, warps=w, warps_per_smsp=bps * w / 4,
                          tflops=round(tf, 3))), flush=True)
for cfg in cfgs:
    for k in (512, 2048):
        ms = min(H.hplk_dgemm_bench(m, m, k, cfg=cfg, reps=5))
        tf = 2 * m * m * k / (ms * 1e-3) / 1e12
        print(json.dumps(dict(cfg=cfg, m=m, k=k, ms=round(ms, 3), tflops=round(tf, 3),
                              frac_dmma=round(tf / peak, 4))), flush=True)

# library context: cuBLAS DGEMM (torch, float64) at the same HPL shape, C -= A B
import torch  # noqa: E402
for k in (512, 2048):
    A = torch.rand(m, k, dtype=torch.float64, device="cuda")
    B = torch.rand(k, m, dtype=torch.float64, device="cuda")
    C = torch.rand(m, m, dtype=torch.float64, device="cuda")
    C.addmm_(A, B, alpha=-1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(5):
        e0.record()
        C.addmm_(A, B, alpha=-1.0)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    tf = 2 * m * m * k / (best * 1e-3) / 1e12
    print(json.dumps(dict(impl="cublas (torch.addmm_ float64)", m=m, k=k, ms=round(best, 3),
                          tflops=round(tf, 3), frac_dmma=round(tf / peak, 4))), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
