"""Chunked bidirectional copies (the bbdg_step_host copy pattern) without kernels."""
import json, time
import torch

K, Np, C = 384000, 220, 40
h_in = torch.empty((4, K, Np), dtype=torch.float32, pin_memory=True)
h_out = torch.empty((4, K, Np), dtype=torch.float32, pin_memory=True)
d_in = torch.empty((4, K, Np), dtype=torch.float32, device="cuda")
d_out = torch.empty((4, K, Np), dtype=torch.float32, device="cuda")
A, B, Cs = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
cs = K // C
out = {}


def run(dep, compute):
    ev = [torch.cuda.Event() for _ in range(C)]
    ev2 = [torch.cuda.Event() for _ in range(C)]
    cur = torch.cuda.current_stream()
    A.wait_stream(cur); B.wait_stream(cur); Cs.wait_stream(cur)
    for i in range(C):
        with torch.cuda.stream(A):
            d_in[:, i * cs:(i + 1) * cs].copy_(h_in[:, i * cs:(i + 1) * cs], non_blocking=True) if False else [
                d_in[F, i * cs:(i + 1) * cs].copy_(h_in[F, i * cs:(i + 1) * cs], non_blocking=True) for F in range(4)]
            ev[i].record(A)
    for i in range(C):
        j = max(0, min(C - 1, i + dep))
        if compute:
            Cs.wait_event(ev[j])
            with torch.cuda.stream(Cs):
                d_out[:, i * cs:(i + 1) * cs].copy_(d_in[:, i * cs:(i + 1) * cs])
            ev2[i].record(Cs)
            B.wait_event(ev2[i])
        else:
            B.wait_event(ev[j])
        with torch.cuda.stream(B):
            for F in range(4):
                h_out[F, i * cs:(i + 1) * cs].copy_(d_out[F, i * cs:(i + 1) * cs], non_blocking=True)
    cur.wait_stream(A); cur.wait_stream(B); cur.wait_stream(Cs)


for name, dep, comp in (("nodep", -10**6, False), ("dep5", 5, False), ("dep5_compute", 5, True)):
    run(dep, comp); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        run(dep, comp)
    torch.cuda.synchronize()
    out[name + "_ms"] = (time.perf_counter() - t0) * 1e3 / 3
print(json.dumps(out))
