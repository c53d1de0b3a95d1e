import re,collections,sys,csv,subprocess
cubin, src_csv, kname, srcfile, moves = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], float(sys.argv[5])
src=open(srcfile).read().splitlines()
call=[i+1 for i,l in enumerate(src) if 'improve_one<W, kDebug>(a, g, s, rec' in l][0]
def fn_of(line):
    for i in range(line-1,-1,-1):
        m=re.search(r'__device__.*?(\w+)\(', src[i]) or re.search(r'__global__.*?(\w+)\(', src[i])
        if m: return m.group(1)
    return None
sass = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-c", "-gi", cubin], capture_output=True, text=True).stdout
amap = {}; on=False; group=[]; cur=None; inner=None
for l in sass.splitlines():
    if l.startswith('.text.'):
        on = kname in l; group=[]; continue
    if not on: continue
    if '## File' in l: group.append(l); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m:
        if group:
            cur=None
            pairs=re.findall(r'"([^"]+)",\s*line\s+(\d+)',group[0])
            inner=pairs[0][0].split('/')[-1]+':'+pairs[0][1]
            for f,n in pairs:
                if f.endswith('improve.cu') and int(n)!=call: cur=int(n); break
        amap[int(m.group(1),16)]=(cur,inner)
        group=[]
rows=list(csv.reader(open(src_csv)))
hdr=rows[1]; data=rows[2:]
ia=hdr.index("Address"); iex=hdr.index("Instructions Executed"); iss=hdr.index("Warp Stall Sampling (All Samples)")
base=int(data[0][ia],16)
byfn=collections.Counter(); stfn=collections.Counter(); byline=collections.Counter(); stline=collections.Counter(); tot=0; tots=0
for r in data:
    a=int(r[ia],16)-base
    ex=int(r[iex] or 0); st=int(r[iss] or 0)
    cur,inner=amap.get(a,(None,None))
    f=fn_of(cur) if cur else 'other:'+str(inner)
    byfn[f]+=ex; stfn[f]+=st; tot+=ex; tots+=st
    if f=='improve_one': byline[cur]+=ex; stline[cur]+=st
print(f'inst/move {tot/moves:.1f}  stall samples {tots}')
for f,v in byfn.most_common(20): print(f'  {f:30s} {v/moves:7.1f} inst/move  {100*stfn[f]/tots:5.1f}% stalls')
print('improve_one lines:')
for k in sorted(byline):
    if byline[k]/moves>=1 or stline[k]/tots>0.01: print(f'  {k} {byline[k]/moves:6.1f} {100*stline[k]/tots:5.1f}%  {src[k-1].strip()[:80]}')
