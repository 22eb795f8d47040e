import csv, io, subprocess, sys, re
out = subprocess.run(["ncu","-i",sys.argv[1],"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
blocks=[]; cur=[]
for ln in out.splitlines():
    if ln.startswith('"Kernel Name"'):
        if cur: blocks.append(cur)
        cur=[ln]
    else: cur.append(ln)
blocks.append(cur)
for b in blocks:
    rows=list(csv.reader(io.StringIO("\n".join(b[1:])))); H={h:i for i,h in enumerate(rows[0])}
    agg={}
    for r in rows[1:]:
        src=r[H["Source"]].strip()
        op=src.split()[0] if not src.startswith("@") else src.split()[1]
        m=re.match(r"(STS\.U16|STS\.128|STS\.64|STS|LDS\.64|LDS\.128|LDS|SYNCS[.\w]*|ATOMS[.\w]*|LDSM|STAS[.\w]*)",op)
        if not m: continue
        k=m.group(1)
        if k=="STS.U16": k += " zero" if "RZ" in src else " val"
        wf=float(r[H["L1 Wavefronts Shared"]] or 0); ex=float(r[H["Instructions Executed"]] or 0)
        a=agg.setdefault(k,[0,0]); a[0]+=wf; a[1]+=ex
    print(b[0][60:140])
    for k,(wf,ex) in sorted(agg.items(), key=lambda x:-x[1][0]):
        print(f"   {k:24s} wf {wf:12.0f} exec {ex:10.0f} wf/inst {wf/max(ex,1):.2f}")
