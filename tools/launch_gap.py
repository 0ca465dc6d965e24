"""Is host submission latency inside the event-timed step? Time the C2 MVM
(stage_dev 3) between events after the L2 flush, with and without a
device-side spin (torch.cuda._sleep) between the flush and the start event
that keeps the GPU busy while the host submits the launch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_12283_b200 as gk  # noqa: E402
from tools.fused_timing import problem  # noqa: E402

op = problem("C2")
nrhs = 32
V = torch.randn(op.size() * nrhs, dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
st = torch.cuda.current_stream()
flush = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
for spin in (0, 20000, 100000, 200000):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in ev:
        flush.sum()
        if spin:
            torch.cuda._sleep(spin)
        a.record(st)
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"spin {spin:7d} cycles: median {np.median(t):6.2f} us  mean {np.mean(t):6.2f}  min {np.min(t):6.2f}", flush=True)
# two back-to-back MVMs inside the events (the second launch needs no SM
# reconfiguration after the flush kernel)
for k in (1, 2, 3):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in ev:
        flush.sum()
        a.record(st)
        for _ in range(k):
            op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"{k} MVMs between events: median {np.median(t):6.2f} us", flush=True)
# flush with a kernel of the same shared-memory carveout: the library's own streaming read
try:
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in ev:
        flush.sum()
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)  # warm the SM config (then L2 holds data)
        flush.sum()
        a.record(st)
        op.stage_dev(3, V.data_ptr(), O.data_ptr(), nrhs, stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"after MVM+flush: median {np.median(t):6.2f} us", flush=True)
except Exception as e:
    print(e)
