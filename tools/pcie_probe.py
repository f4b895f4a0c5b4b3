"""PCIe copy-bandwidth probe (pinned host <-> device), one direction at a time
and both directions concurrently, at the e2e transfer size (128^3: 51.5 MB).
Output: one JSON line.  Used to bound bench.py's e2e."""
import json
import sys

import torch

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 51520536
n = nb // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda").fill_(2.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
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
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def both_split(k):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    step = (n + k - 1) // k

    def f():
        cur = torch.cuda.current_stream()
        for st in ss:
            st.wait_stream(cur)
        for i in range(k):
            lo, hi = i * step, min(n, (i + 1) * step)
            with torch.cuda.stream(ss[i]):
                d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            with torch.cuda.stream(ss[k + i]):
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
        for st in ss:
            cur.wait_stream(st)
    return f


t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
split = {k: timed(both_split(k)) for k in (2, 4, 8)}
print(json.dumps({"bytes": nb, "h2d_ms": t_h2d, "d2h_ms": t_d2h, "both_ms": t_both,
                  "h2d_gbs": nb / t_h2d / 1e6, "d2h_gbs": nb / t_d2h / 1e6,
                  "both_gbs_per_dir": nb / t_both / 1e6,
                  "both_split_gbs_per_dir": {k: nb / v / 1e6 for k, v in split.items()}}))
