"""Where does the e2e step's time go? Times spmv_create from pinned host COO
alone, the device-resident power loop alone, and both concurrently on two
streams/threads (c2)."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402
from paper_2302_05662_b200.dist import Layout, native_power_iteration  # noqa: E402

coo = si.config_device("c2")
n = coo.rows
hr, hc, hv = (t.cpu().pin_memory() for t in (coo.row, coo.col, coo.val))
E = 100
layout = Layout.from_bounds(np.array([0, n]))


def create(st):
    with torch.cuda.stream(st):
        h = P.spmv_create(coo.rows, coo.cols, hr.numpy(), hc.numpy(), hv.numpy(), stream=st)
        st.synchronize()
    return h


def power(h, st, bufs, x):
    with torch.cuda.stream(st):
        native_power_iteration(h, layout, 0, x, bufs, E)
        st.synchronize()


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x = si.vector_device(n)
bufs = {"cur": torch.zeros(n, dtype=torch.float64, device="cuda"), "nxt": torch.zeros(n, dtype=torch.float64, device="cuda"),
        "chunk": torch.zeros(1, dtype=torch.float64, device="cuda"), "sums": torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")}
hp = create(s2)
P.spmv_features(hp)
P.spmv_convert(hp, P.FMT_ELL, index16=1)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); h = create(s1); t1 = time.perf_counter(); P.spmv_destroy(h)
    print(f"create from host alone: {1e3 * (t1 - t0):.2f} ms ({(hr.numel() * 16) / (t1 - t0) / 1e9:.1f} GB/s)")
    t0 = time.perf_counter(); power(hp, s2, bufs, x); t1 = time.perf_counter()
    print(f"power loop alone: {1e3 * (t1 - t0):.2f} ms")
    t0 = time.perf_counter(); a = torch.empty(hr.numel() * 4, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s1):
        a[:hr.numel()].copy_(hr, non_blocking=True); a[hr.numel():2 * hr.numel()].copy_(hc, non_blocking=True)
        b = torch.empty(hv.numel(), dtype=torch.float64, device="cuda"); b.copy_(hv, non_blocking=True)
        s1.synchronize()
    t1 = time.perf_counter()
    print(f"torch H2D of the same bytes: {1e3 * (t1 - t0):.2f} ms")
    res = {}

    def tc():
        t = time.perf_counter(); h = create(s1); res["c"] = time.perf_counter() - t; P.spmv_destroy(h)

    def tp():
        t = time.perf_counter(); power(hp, s2, bufs, x); res["p"] = time.perf_counter() - t
    t0 = time.perf_counter()
    th = [threading.Thread(target=tc), threading.Thread(target=tp)]
    [t.start() for t in th]; [t.join() for t in th]
    t1 = time.perf_counter()
    print(f"concurrent: total {1e3 * (t1 - t0):.2f} ms, create {1e3 * res['c']:.2f}, power {1e3 * res['p']:.2f}")

# ---- the bench's whole e2e step, serial vs two lanes, with per-phase host times
x0h = x.cpu().pin_memory()


def step(st, bufs_, yh, lock, log):
    with torch.cuda.stream(st):
        t = [time.perf_counter()]
        xd = torch.empty_like(x)
        with lock:
            h = P.spmv_create(coo.rows, coo.cols, hr.numpy(), hc.numpy(), hv.numpy(), stream=st)
            xd.copy_(x0h, non_blocking=True)
        t.append(time.perf_counter())
        P.spmv_features(h)
        t.append(time.perf_counter())
        P.spmv_convert(h, P.FMT_ELL, index16=1)
        t.append(time.perf_counter())
        native_power_iteration(h, layout, 0, xd, bufs_, E)
        yh.copy_(bufs_["cur"], non_blocking=True)
        t.append(time.perf_counter())
        st.synchronize()
        t.append(time.perf_counter())
        P.spmv_destroy(h)
        t.append(time.perf_counter())
        log.append([round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])])


lock = threading.Lock()
bufs2 = {k: torch.zeros_like(v) for k, v in bufs.items()}
yh1 = torch.empty(n, dtype=torch.float64).pin_memory()
yh2 = torch.empty(n, dtype=torch.float64).pin_memory()
for mode in ("serial", "two lanes", "serial", "two lanes"):
    logs = [[], []]
    t0 = time.perf_counter()
    if mode == "serial":
        for _ in range(8):
            step(s1, bufs, yh1, lock, logs[0])
    else:
        th = [threading.Thread(target=lambda i=i: [step((s1, s2)[i], (bufs, bufs2)[i], (yh1, yh2)[i], lock, logs[i])
                                                   for _ in range(4)]) for i in range(2)]
        [t.start() for t in th]; [t.join() for t in th]
    t1 = time.perf_counter()
    print(f"{mode}: {1e3 * (t1 - t0) / 8:.2f} ms per step; phases [create, features, convert, launch, sync, destroy]:")
    for i, lg in enumerate(logs):
        for r in lg[:3]:
            print("   lane", i, r)
