import ctypes as C, os, sys, torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbw.so"))
nbytes = int(54.5e6) // 4096 * 4096
buf = torch.ones(nbytes, dtype=torch.uint8, device="cuda")
out = torch.zeros(4, dtype=torch.int32, device="cuda")
fw = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
fr = torch.ones(256 << 20, dtype=torch.uint8, device="cuda").view(torch.int64)
st = torch.cuda.current_stream().cuda_stream
def timeit(fn, mode):
    ts = []
    for i in range(30):
        fw.zero_()
        if mode == "wr":
            fr.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort(); return ts[len(ts) // 2]
for mode in ("w", "wr"):
    for blocks, threads in ((148 * 4, 512), (148 * 8, 256), (148 * 16, 256), (148 * 32, 256)):
        t = timeit(lambda: L.run_read(C.c_void_p(buf.data_ptr()), C.c_size_t(nbytes), blocks, threads, C.c_void_p(out.data_ptr()), C.c_void_p(st)), mode)
        print(f"flush {mode} ldg blocks {blocks} x {threads}: {t:.1f} us = {nbytes / t / 1e3:.0f} GB/s", flush=True)
    for chunk in (8192, 12288):
        t = timeit(lambda: L.run_bulk(C.c_void_p(buf.data_ptr()), C.c_size_t(nbytes), 148, chunk, C.c_void_p(out.data_ptr()), C.c_void_p(st)), mode)
        print(f"flush {mode} bulk chunk {chunk} x16 ring: {t:.1f} us = {nbytes / t / 1e3:.0f} GB/s", flush=True)
