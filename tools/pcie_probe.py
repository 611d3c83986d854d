"""Host<->device copy bandwidth on this box: pinned H2D / D2H alone and both
directions at once, one or two streams per direction (e2e bound of bench.py)."""
import torch

N = 512 << 20  # bytes per tensor (one bf16 (1,16,131072,128) tensor)
K = 4          # tensors per direction per step (q,k,v,dO in; out,dq,dk,dv out)
dev = [torch.empty(N, dtype=torch.uint8, device="cuda") for _ in range(2 * K)]
host_in = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(K)]
host_out = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(K)]


def run(h2d: bool, d2h: bool, nstreams: int, reps: int = 3) -> float:
    streams = [torch.cuda.Stream() for _ in range(2 * nstreams)]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        for i in range(K):
            if h2d:
                s = streams[i % nstreams]
                s.wait_event(a)
                with torch.cuda.stream(s):
                    dev[i].copy_(host_in[i], non_blocking=True)
            if d2h:
                s = streams[nstreams + i % nstreams]
                s.wait_event(a)
                with torch.cuda.stream(s):
                    host_out[i].copy_(dev[K + i], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return reps * K * N / (ms / 1e3) / 1e9


for ns in (1, 2):
    print(f"streams/dir={ns}: H2D {run(True, False, ns):.1f} GB/s  D2H {run(False, True, ns):.1f} GB/s  "
          f"both {run(True, True, ns):.1f} GB/s per direction")
