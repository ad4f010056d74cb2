"""Host-link probe: pinned H2D / D2H bandwidth alone and concurrently (both
directions at once on two streams), for the e2e roofline. Prints one JSON line.

    python tools/pcie_probe.py [--gib 2]
"""
import argparse
import json

import torch


def timed(fn, dev):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    n = a.gib << 30
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_src = torch.empty(n, dtype=torch.uint8, device=dev)
    d_dst = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}
    for name, fn in {"h2d": lambda: d_dst.copy_(h_src, non_blocking=True),
                     "d2h": lambda: h_dst.copy_(d_src, non_blocking=True)}.items():
        out[name] = max(n / timed(fn, dev) / 1e9 for _ in range(3))

    def both():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            d_dst.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_src, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s1)
        torch.cuda.current_stream(dev).wait_stream(s2)

    t = min(timed(both, dev) for _ in range(3))
    out["bidir_each"] = n / t / 1e9
    out["bidir_total"] = 2 * n / t / 1e9
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
