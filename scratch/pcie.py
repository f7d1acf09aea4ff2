"""scratch: pinned H2D / D2H bandwidth alone and concurrently (not part of the product)."""
import torch
n = 4 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def ev(): return torch.cuda.Event(enable_timing=True)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) * 1e3 / reps
print("H2D 4MB", t(lambda: d1.copy_(h1, non_blocking=True)))
print("D2H 4MB", t(lambda: h2.copy_(d2, non_blocking=True)))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
print("both concurrently", t(both))
for ch in (2, 4, 8, 16):
    c = n // ch
    def chunked():
        for i in range(ch): d1[i*c:(i+1)*c].copy_(h1[i*c:(i+1)*c], non_blocking=True)
    print("H2D in", ch, "chunks", t(chunked))
