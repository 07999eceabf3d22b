"""PCIe copy ceiling for the C2 e2e leg: pinned host <-> HBM bandwidth, each direction
alone and both at once (two streams), with the same byte counts as one C2 e2e step
(H2D 2.17 GB of variates + filter result, D2H 2.15 GB of paths).  Device-timed with
CUDA events; prints one JSON line (profiles/r1e_pcie_copy.json)."""
import json
import torch

H2D, D2H = 2168488264, 2147516416
n_in, n_out = H2D // 8, D2H // 8
hin = torch.empty(n_in, dtype=torch.float64, pin_memory=True)
hout = torch.empty(n_out, dtype=torch.float64, pin_memory=True)
din = torch.empty(n_in, dtype=torch.float64, device="cuda")
dout = torch.zeros(n_out, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def h2d():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
print(json.dumps({
    "h2d_bytes": H2D, "d2h_bytes": D2H,
    "h2d_ms": t_in, "h2d_GBps": H2D / t_in / 1e6,
    "d2h_ms": t_out, "d2h_GBps": D2H / t_out / 1e6,
    "both_ms": t_both, "both_GBps_total": (H2D + D2H) / t_both / 1e6,
    "note": "C2 e2e step floor = both_ms (copies alone, no sampling)"}))
