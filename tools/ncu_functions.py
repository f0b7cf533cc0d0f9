#!/usr/bin/env python
"""Per-function view of an ncu --set full capture: executed warp instructions
and stall samples attributed to the device function (file:function) each
source line belongs to.

    python tools/ncu_functions.py gpurun_out/x.ncu-rep <frames in the launch>
"""
import subprocess, csv, io, collections, re, sys
rep=sys.argv[1]; nfr=float(sys.argv[2])
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
def fl(x):
    try: return float(x.replace(',',''))
    except: return 0.0
inst=collections.Counter(); samp=collections.Counter()
fname=line='?'; head=None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0]=="File Path": fname=row[1].split('/')[-1]; continue
    if row[0]=="Line No": head=row; continue
    if head is None or len(row)<len(head): continue
    if row[0]: line=int(row[0]); continue
    d=dict(zip(head[4:],row[4:]))
    inst[(fname,line)]+=fl(d["Instructions Executed"]); samp[(fname,line)]+=fl(d["Warp Stall Sampling (All Samples)"])
base='paper_2604_02266_b200/csrc/'
funcs={}
for fn in ['sscga_tm.cu','cg.cuh','common.cuh','demod.cuh','sscga.cu']:
    src=open(base+fn).read().splitlines(); lst=[]
    for i,l in enumerate(src,1):
        m2=re.search(r'(?:__forceinline__|__launch_bounds__\([\w\(\), ]*\))\s+[\w<>:&,\s\*]*?(\w+)\(', l)
        if m2: lst.append((i,m2.group(1)))
    funcs[fn]=(lst,src)
def func_of(f,line):
    if f not in funcs: return f
    name='?'
    for i,n in funcs[f][0]:
        if i<=line: name=n
    return f+':'+name
agg=collections.Counter(); aggs=collections.Counter()
for (f,l),n in inst.items():
    k=func_of(f,l); agg[k]+=n; aggs[k]+=samp[(f,l)]
ti=sum(agg.values()); ts=sum(aggs.values())
print("total inst per frame", ti/nfr)
for k,v in agg.most_common(30): print(f"{100*v/ti:6.1f}% inst {100*aggs[k]/ts:6.1f}% samp  {v/nfr:9.0f}/frame  {k}")
