"""Host<->device copy bandwidth from pinned memory: one stream vs two (diagnostic)."""
import torch
n = 512 << 20   # 512 MiB per buffer (one bf16 q/k/v/dy tensor of configs[1])
hs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(4)]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(4)]
st = [torch.cuda.Stream() for _ in range(4)]
def run(nstreams, d2h=False):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(4):
        s = st[i % nstreams]
        s.wait_event(e0)
        with torch.cuda.stream(s):
            if d2h:
                hs[i].copy_(ds[i], non_blocking=True)
            else:
                ds[i].copy_(hs[i], non_blocking=True)
    for i in range(nstreams):
        torch.cuda.current_stream().wait_stream(st[i])
    e1.record()
    torch.cuda.synchronize()
    return 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
for k in (1, 2, 4):
    run(k); print(f"H2D {k} stream(s): {run(k):.1f} GB/s   D2H: {run(k, True):.1f} GB/s")
# both directions at once
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(2):
    st[i].wait_event(e0)
    with torch.cuda.stream(st[i]):
        ds[i].copy_(hs[i], non_blocking=True)
    st[2 + i].wait_event(e0)
    with torch.cuda.stream(st[2 + i]):
        hs[2 + i].copy_(ds[2 + i], non_blocking=True)
for i in range(4):
    torch.cuda.current_stream().wait_stream(st[i])
e1.record()
torch.cuda.synchronize()
print(f"duplex: {4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s total")
