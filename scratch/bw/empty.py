import ctypes as C, os, torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libempty.so"))
st = torch.cuda.current_stream().cuda_stream
def ev(): return torch.cuda.Event(enable_timing=True)
def t(fn, n=30):
    ts = []
    for i in range(n):
        torch.cuda._sleep(1000000); s, e = ev(), ev(); s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort(); return ts[n // 2], ts[0]
print("events only", t(lambda: None))
for b, th, sm in ((1, 32, 0), (148, 448, 0), (148, 448, 210 * 1024), (2368, 256, 0), (148, 1024, 0)):
    L.run_empty(b, th, sm, C.c_void_p(st))
    print(b, th, sm, t(lambda: L.run_empty(b, th, sm, C.c_void_p(st))))
# 10 back-to-back empties between events
print("10x 148x448 smem", t(lambda: [L.run_empty(148, 448, 210 * 1024, C.c_void_p(st)) for _ in range(10)]))
