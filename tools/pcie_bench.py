"""Pinned host <-> device copy rates, one direction and both at once
(development tool: the ceiling of bench.py's e2e numbers)."""
import json

import torch


def main():
    nb = 1 << 30
    h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
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

    out["h2d_GBs"] = nb / timed(lambda: d_in.copy_(h_in, non_blocking=True)) / 1e6
    out["d2h_GBs"] = nb / timed(lambda: h_out.copy_(d_out, non_blocking=True)) / 1e6
    cur = torch.cuda.current_stream()

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    ms = timed(both)
    out["duplex_ms_1GB_each_way"] = ms
    out["duplex_GBs_each_way"] = nb / ms / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
