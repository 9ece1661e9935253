"""PCIe copy ceilings for the e2e leg: pinned host <-> HBM, 33.5 MB per
direction (one C2 window's actions in and dL/d(actions) out), H2D alone,
D2H alone and both at once on two streams; chunked variants."""
import time

import torch

NB = 32 * 65536 * 4 * 4  # bytes: T x N x A fp32
n = NB // 4
h_in = [torch.randn(n).pin_memory() for _ in range(2)]
h_out = [torch.empty(n).pin_memory() for _ in range(2)]
d = [torch.empty(n, device="cuda") for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(kind, reps=40, chunks=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(reps):
        c = n // chunks
        for j in range(chunks):
            sl = slice(j * c, (j + 1) * c)
            if kind in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d[k % 2][sl].copy_(h_in[k % 2][sl], non_blocking=True)
            if kind in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out[k % 2][sl].copy_(d[2 + k % 2][sl], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return {"ms_per_window": dt * 1e3, "GBps_per_direction": NB / dt / 1e9}


for kind in ("h2d", "d2h", "both"):
    for ch in (1, 4):
        run(kind, 5, ch)
        print(kind, "chunks", ch, run(kind, 40, ch))

# the same bidirectional copies while an HBM-heavy kernel stream runs beside
# them (the e2e leg's situation: window kernels at ~4 TB/s between the copies)
big = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
s3 = torch.cuda.Stream()


def run_loaded(reps=40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s3):
        for _ in range(reps * 4):
            big.mul_(1.0000001)  # 2 x 256 MB per launch, ~0.08 ms
    for k in range(reps):
        with torch.cuda.stream(s1):
            d[k % 2].copy_(h_in[k % 2], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[k % 2].copy_(d[2 + k % 2], non_blocking=True)
    s1.synchronize()
    s2.synchronize()
    dt = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    return {"ms_per_window": dt * 1e3, "GBps_per_direction": NB / dt / 1e9}


run_loaded(5)
print("both + HBM load", run_loaded(40))
