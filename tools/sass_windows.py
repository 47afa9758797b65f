"""Per-window summary of an ncu --page source --csv --print-source sass export:
    python tools/sass_windows.py KERNEL_INDEX WINDOW CSV"""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[3] if len(sys.argv) > 3 else '/tmp/src_sass.csv')))
kern = [i for i,r in enumerate(rows) if r and r[0]=='Kernel Name']
which = int(sys.argv[1]) if len(sys.argv)>1 else 0
W = int(sys.argv[2]) if len(sys.argv)>2 else 300
start = kern[which]+2
end = kern[which+1] if which+1 < len(kern) else len(rows)
hdr = rows[kern[which]+1]
ci = {h:i for i,h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
body = rows[start:end]
tot = sum(int(r[ci['Warp Stall Sampling (All Samples)']] or 0) for r in body)
print('kernel', rows[kern[which]][1], 'instructions', len(body), 'samples', tot)
def op(r):
    s = r[1].strip()
    s = re.sub(r'^@!?U?P\w+\s+','',s)
    return s.split()[0] if s else ''
for w0 in range(0, len(body), W):
    chunk = body[w0:w0+W]
    smp = sum(int(r[ci['Warp Stall Sampling (All Samples)']] or 0) for r in chunk)
    ops = collections.Counter(op(r).split('.')[0] for r in chunk)
    st = collections.Counter()
    for r in chunk:
        for h in stalls:
            v = r[ci[h]]
            if v and v != '0': st[h[6:]] += int(v)
    top = ', '.join(f'{k}:{v*100//max(1,smp)}%' for k,v in st.most_common(4))
    keyops = ' '.join(f'{k}{ops[k]}' for k in ('DMMA','DFMA','DMUL','DADD','LDS','STS','LDG','STG','LDGSTS','BAR','UBLKCP','SYNCS','LDC','SHFL') if ops[k])
    print(f'{w0:6d} {smp*100/tot:5.1f}% | {keyops} | {top}')
