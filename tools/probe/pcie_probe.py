"""PCIe copy bandwidth probe (not product): pinned host <-> device, one or two streams per
direction, and both directions at once; CUDA events, 1 GiB per direction."""
import torch
dev = torch.device("cuda:0")
n = 1 << 30
h_in = [torch.empty(n // 2, dtype=torch.uint8).pin_memory() for _ in range(2)]
h_out = [torch.empty(n // 2, dtype=torch.uint8).pin_memory() for _ in range(2)]
d_in = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(2)]
d_out = [torch.ones(n // 2, dtype=torch.uint8, device=dev) for _ in range(2)]
ss = [torch.cuda.Stream(dev) for _ in range(4)]
def run(h2d_streams, d2h_streams, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for st in ss:
            st.wait_event(s)
        evs = []
        for i in range(2):
            if h2d_streams:
                st = ss[i % h2d_streams]
                with torch.cuda.stream(st):
                    d_in[i].copy_(h_in[i], non_blocking=True)
            if d2h_streams:
                st = ss[2 + i % d2h_streams]
                with torch.cuda.stream(st):
                    h_out[i].copy_(d_out[i], non_blocking=True)
        for st in ss:
            ev = torch.cuda.Event(); ev.record(st); torch.cuda.current_stream().wait_event(ev)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    moved = n * ((1 if h2d_streams else 0) + (1 if d2h_streams else 0))
    return f"{best:.1f} ms, {moved / best / 1e6:.1f} GB/s"
print("H2D 1 stream ", run(1, 0)); print("H2D 2 streams", run(2, 0))
print("D2H 1 stream ", run(0, 1)); print("D2H 2 streams", run(0, 2))
print("both 1+1     ", run(1, 1)); print("both 2+2     ", run(2, 2))
