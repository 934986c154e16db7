"""Raw PCIe copy bandwidth (development): pinned host <-> HBM, one direction
and both at once on two streams, 1 GiB transfers, CUDA events."""
import json
import torch

nb = 1 << 30
h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


out = {"h2d_gbs": nb / timed(h2d) / 1e9, "d2h_gbs": nb / timed(d2h) / 1e9, "both_gbs_total": 2 * nb / timed(both) / 1e9}
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
