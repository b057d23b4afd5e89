import torch, time
n = 128 * 2**20 // 8
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
hin = torch.randn(n, dtype=torch.float64).pin_memory()
s = [torch.cuda.Stream() for _ in range(4)]
def run(k, direction="d2h"):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    chunk = n // k
    evs = []
    for i in range(k):
        s[i].wait_event(e0)
        with torch.cuda.stream(s[i]):
            if direction == "d2h":
                h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
            elif direction == "h2d":
                d[i*chunk:(i+1)*chunk].copy_(hin[i*chunk:(i+1)*chunk], non_blocking=True)
            ev = torch.cuda.Event(); ev.record(); evs.append(ev)
    for ev in evs: torch.cuda.current_stream().wait_event(ev)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return 128 / 1024 / (ms / 1e3), ms
for direction in ("d2h", "h2d"):
    for k in (1, 2, 4, 1, 2, 4):
        gbs, ms = run(k, direction)
        print(direction, "streams", k, f"{ms:.2f} ms  {gbs:.1f} GB/s")
# concurrent h2d + d2h
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
s[0].wait_event(e0); s[1].wait_event(e0)
with torch.cuda.stream(s[0]): h.copy_(d, non_blocking=True)
d2 = torch.empty_like(d)
with torch.cuda.stream(s[1]): d2.copy_(hin, non_blocking=True)
torch.cuda.current_stream().wait_stream(s[0]); torch.cuda.current_stream().wait_stream(s[1])
e1.record(); torch.cuda.synchronize()
print("bidirectional", f"{e0.elapsed_time(e1):.2f} ms for 128 MB each way")
