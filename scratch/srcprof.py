import csv,re,collections,sys
want=sys.argv[1]; units=int(sys.argv[2]) if len(sys.argv)>2 else 4096
rows=list(csv.reader(open('/tmp/src.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='Address'][0]
hdr=rows[hi]; iA=hdr.index('Address'); iE=hdr.index('Instructions Executed'); iW=hdr.index('Warp Stall Sampling (All Samples)')
data=[(int(r[iA],16), float(r[iE] or 0), float(r[iW] or 0)) for r in rows[hi+1:] if len(r)>iE and r[iA].startswith('0x')]
base=min(a for a,_,_ in data)
cur=None; line=None; addr2line={}
for l in open('/tmp/cub/all.sass'):
    m=re.match(r'\s*\.section\s+\.text\.(\S+)',l)
    if m: cur=m.group(1).split(',')[0]; continue
    if cur!=want: continue
    m=re.search(r'//## File "(.*)", line (\d+)',l)
    if m: line=(m.group(1).split('/')[-1],int(m.group(2))); continue
    m=re.match(r'\s+/\*([0-9a-f]+)\*/',l)
    if m: addr2line[int(m.group(1),16)]=line
cnt=collections.Counter(); smp=collections.Counter()
for a,e,w in data: cnt[addr2line.get(a-base)]+=e; smp[addr2line.get(a-base)]+=w
print('total/tile', sum(cnt.values())/units, 'samples', sum(smp.values()))
src=open('paper_2605_08317_b200/csrc/decode_mma.cu').read().split('\n')
for k,v in cnt.most_common(int(sys.argv[3]) if len(sys.argv)>3 else 30):
    txt = src[k[1]-1].strip()[:90] if k and k[0]=='decode_mma.cu' else str(k)
    print(f"{v/units:8.1f} {smp[k]:6.0f} {k[1] if k else ''} {txt}")
