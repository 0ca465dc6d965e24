"""K_UU MVM: the reference's circulant-embedding FFT route (dski.cpp:146-166)
measured with cuFFT (torch.fft, batched over RHS: the best library FFT on this
GPU, an upper bound on what an in-house FFT would reach) against this build's
Kronecker-Toeplitz DMMA mode products (gk stage 1), at C2 (100², 32 RHS),
C3 (48³, 17 RHS) and C4 (400², 1 RHS). Same inputs; also checks that both
give the same product (the FFT's spectrum is real: dski.cpp:128-132)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream()
flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def tm(fn, reps=30):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.sum()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


for cfg, ell, nodes, nrhs in ((2, 0.2, 100, 32), (3, 0.3, 48, 17), (4, 0.02, 400, 1)):
    X, *_ = gk.make_dataset(cfg, 0)
    grid = gk.Grid.cover(X, 1e-4, 3, nodes)
    op = gk.DskiOperator(gk.KernelSpec(ell, 1.0), grid, X, (1e-2, 1e-2))
    dims = [int(x) for x in grid.dims]
    M = int(np.prod(dims))
    # spectrum of the circulant embedding (e_j = 2(m_j - 1), wrapped offsets)
    emb = [2 * (m - 1) for m in dims]
    axes = []
    for j, (m, e) in enumerate(zip(dims, emb)):
        idx = np.arange(e)
        off = np.where(idx <= e // 2, idx, idx - e) * grid.spacing[j]
        axes.append(np.exp(-0.5 * off ** 2 / ell ** 2))
    slice_ = axes[0]
    for a in axes[1:]:
        slice_ = np.multiply.outer(slice_, a)
    spec = torch.from_numpy(np.fft.rfftn(slice_).real.copy()).to(dev)
    U = torch.randn([nrhs] + dims, dtype=torch.float64, device=dev)

    def fft_mvm():
        P = torch.zeros([nrhs] + emb, dtype=torch.float64, device=dev)
        P[(slice(None),) + tuple(slice(0, m) for m in dims)] = U
        Fh = torch.fft.rfftn(P, dim=tuple(range(1, len(dims) + 1)))
        Fh *= spec
        W = torch.fft.irfftn(Fh, s=emb, dim=tuple(range(1, len(dims) + 1)))
        return W[(slice(None),) + tuple(slice(0, m) for m in dims)]

    # the library's K_UU on the same block: internal grid layout is node-major, RHS innermost
    Ui = U.reshape(nrhs, M).t().contiguous()
    Wi = torch.empty_like(Ui)

    def dmma_mvm():
        op.stage_dev(1, Ui.data_ptr(), Wi.data_ptr(), nrhs, stream=st.cuda_stream)

    t_fft = tm(fft_mvm)
    t_dmma = tm(dmma_mvm)
    Wf = fft_mvm().reshape(nrhs, M).t()
    dmma_mvm()
    torch.cuda.synchronize()
    err = float((Wf - Wi).norm() / Wi.norm())
    print(f"C{cfg} grid {dims} emb {emb} nrhs {nrhs}: cuFFT circulant {t_fft:8.1f} us   "
          f"Toeplitz DMMA {t_dmma:8.1f} us   ratio {t_fft / t_dmma:5.2f}   rel diff {err:.1e}", flush=True)
