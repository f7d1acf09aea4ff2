"""tools: summarise an ncu report of the decode kernel (metrics, stalls, per-line instructions)."""
import csv, collections, io, re, subprocess, sys
rep = sys.argv[1]
units = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
nlines = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
for w in ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size',
          'launch__block_size', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
          'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
          'sm__cycles_elapsed.avg.per_second', 'smsp__cycles_active.avg', 'sm__cycles_elapsed.avg']:
    if w in h:
        print(f"{w:60s} {v[h.index(w)][:90]}")
ie = h.index('smsp__inst_executed.sum')
print("instructions per unit", float(v[ie].replace(',', '')) / units)
st = [(x, v[i]) for i, x in enumerate(h) if x.startswith('smsp__pcsamp_warps_issue_stalled') and not x.endswith('not_issued')]
st = sorted(((float(b.replace(',', '')) if b else 0, a.replace('smsp__pcsamp_warps_issue_stalled_', '')) for a, b in st), reverse=True)[:10]
print("stalls:", ", ".join(f"{n}={int(c)}" for c, n in st))
kname = v[h.index('Kernel Name')]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
hdr = rows[hi]
iA, iE, iW, iS = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Source')
data = [(int(r[iA], 16), float(r[iE] or 0), float(r[iW] or 0), r[iS].strip()) for r in rows[hi + 1:] if len(r) > iE and r[iA].startswith('0x')]
ops = collections.Counter()
for a, e, w, s in data:
    op = s.split()[0] if s else '?'
    if op.startswith('@'):
        op = s.split()[1]
    ops[op.split('.')[0]] += e
print("opcodes/unit:", ", ".join(f"{k}={v / units:.0f}" for k, v in ops.most_common(24)))
if len(sys.argv) > 4:  # per-line with a cubin disassembly and mangled name
    sass, want = sys.argv[4], sys.argv[5]
    base = min(a for a, *_ in data)
    cur = line = None
    a2l = {}
    for l in open(sass):
        m = re.match(r'\s*\.section\s+\.text\.(\S+)', l)
        if m:
            cur = m.group(1).split(',')[0]
            continue
        if cur != want:
            continue
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m:
            line = (m.group(1).split('/')[-1], int(m.group(2)))
            continue
        m = re.match(r'\s+/\*([0-9a-f]+)\*/', l)
        if m:
            a2l[int(m.group(1), 16)] = line
    cnt, smp = collections.Counter(), collections.Counter()
    for a, e, w, s in data:
        cnt[a2l.get(a - base)] += e
        smp[a2l.get(a - base)] += w
    srcl = open('paper_2605_08317_b200/csrc/decode_mma.cu').read().split('\n')
    for k, c in cnt.most_common(nlines):
        txt = srcl[k[1] - 1].strip()[:88] if k and k[0] == 'decode_mma.cu' else str(k)
        print(f"{c / units:7.1f} {smp[k]:6.0f} {k[1] if k else ''} {txt}")
