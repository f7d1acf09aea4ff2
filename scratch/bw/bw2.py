"""scratch: HBM read floor vs size and timing method (not part of the product)."""
import ctypes as C, os, torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbw.so"))
big = torch.ones(4 << 30, dtype=torch.uint8, device="cuda")
out = torch.zeros(4, dtype=torch.int32, device="cuda")
fw = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def rd(off, nbytes):
    L.run_read(C.c_void_p(big.data_ptr() + off), C.c_size_t(nbytes), 148 * 16, 256, C.c_void_p(out.data_ptr()), C.c_void_p(st))
def ev():
    return torch.cuda.Event(enable_timing=True)
for nbytes in (0, 4096):
    ts = []
    for i in range(20):
        torch.cuda._sleep(2000000); s, e = ev(), ev(); s.record(); rd(0, nbytes); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort(); fw.zero_(); ts2=[]
    print(f"tiny read {nbytes} B: {ts[10]:.2f} us", flush=True)
for mb in (13, 27, 54, 108, 216, 432, 864):
    nbytes = (mb << 20)
    ts = []
    for i in range(20):
        torch.cuda._sleep(2000000); fw.zero_(); s, e = ev(), ev(); s.record(); rd(0, nbytes); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort(); a = ts[10]
    nrot = min(max(2, (1 << 30) // nbytes + 1), (4 << 30) // nbytes)
    K = 40
    es = [ev() for _ in range(K + 1)]
    for i in range(5): rd((i % nrot) * nbytes, nbytes)
    torch.cuda._sleep(5000000)
    es[0].record()
    for i in range(K):
        rd(((i + 5) % nrot) * nbytes, nbytes); es[i + 1].record()
    torch.cuda.synchronize()
    per = sorted(es[i].elapsed_time(es[i + 1]) * 1e3 for i in range(K))
    tot = es[0].elapsed_time(es[K]) * 1e3 / K
    print(f"{mb:4d} MB: flushed {a:7.1f} us ({nbytes/a/1e3:5.0f} GB/s) | back-to-back rot x{nrot}: {tot:7.1f} us/launch ({nbytes/tot/1e3:5.0f} GB/s), median per-launch {per[K//2]:.1f}", flush=True)
# zero-byte launch right after a flush
ts = []
for i in range(20):
    torch.cuda._sleep(2000000); fw.zero_(); s, e = ev(), ev(); s.record(); rd(0, 0); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
ts.sort(); print(f"flushed 0-byte launch: {ts[10]:.2f} us", flush=True)
