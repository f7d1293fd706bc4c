"""Pinned host<->device copy bandwidth on this box: H2D, D2H, and both at once (two streams).

    python tools/pcie_bw.py [--mb 338]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=338)
    a = ap.parse_args()
    n = a.mb << 20
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def h2d():
        d1.copy_(h1, non_blocking=True)

    def d2h():
        h2.copy_(d2, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
        ms = timed(fn)
        out[name + "_gbs"] = (2 if name == "both" else 1) * n / (ms * 1e-3) / 1e9
    out["mb"] = a.mb
    print(json.dumps(out))


if __name__ == "__main__":
    main()
