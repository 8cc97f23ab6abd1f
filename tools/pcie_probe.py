import torch, time
n = 960_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for it in range(3):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("H2D one copy GB/s", n / s.elapsed_time(e) / 1e6)
    s.record(); h.copy_(d, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("D2H one copy GB/s", n / s.elapsed_time(e) / 1e6)
# chunked on two streams
st = [torch.cuda.Stream() for _ in range(2)]
c = 64 << 20
s.record()
for i, o in enumerate(range(0, n, c)):
    with torch.cuda.stream(st[i % 2]):
        d[o:o+c].copy_(h[o:o+c], non_blocking=True)
for x in st: torch.cuda.current_stream().wait_stream(x)
e.record(); torch.cuda.synchronize()
print("H2D 2-stream chunks GB/s", n / s.elapsed_time(e) / 1e6)
# simultaneous H2D + D2H
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s.record()
with torch.cuda.stream(st[0]): d.copy_(h, non_blocking=True)
with torch.cuda.stream(st[1]): h2.copy_(d2, non_blocking=True)
for x in st: torch.cuda.current_stream().wait_stream(x)
e.record(); torch.cuda.synchronize()
print("duplex both dirs ms", s.elapsed_time(e))
# 256 MB tiles back to back on one stream (run_streamed's pattern)
c = 256 << 20
for it in range(2):
    s.record()
    for o in range(0, n, c):
        d[o:o+c].copy_(h[o:o+c], non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("H2D 256MB tiles one stream GB/s", n / s.elapsed_time(e) / 1e6)
# same with an HBM-bound kernel running beside it (both on side streams)
big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(ks):
    for _ in range(40): big.add_(1)
with torch.cuda.stream(cs):
    s.record(cs)
    for o in range(0, n, c):
        d[o:o+c].copy_(h[o:o+c], non_blocking=True)
    e.record(cs)
torch.cuda.synchronize()
print("H2D 256MB tiles beside HBM load GB/s", n / s.elapsed_time(e) / 1e6)
