import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
src=open('/root/repo/paper_2404_15217_b200/csrc/pf_multicrop.cu').read().split('\n')
# phases by markers in source
marks=[]
for i,l in enumerate(src,1):
    for key,name in [('// adjust_hue','hue'),('// Packed FP32 pairs','f2ops'),('// RandomResizedCrop resample tables','tables'),('// 12 floats','load12'),('// Horizontal RRC pass','rrc_h'),('// pack four bytes','pack'),('// Vertical RRC pass','rrc_v'),('// The fused kernel','k_setup'),('// ---- 1. gather','stage'),('// horizontal pass ww','hpass'),('// vertical pass ->','vpass'),('// ---- 2. ColorJitter','jitter'),('// ---- 3/4. blur','epi_noblur'),('// separable 9-tap blur','blur'),('}  // namespace pf','tail')]:
        if key in l: marks.append((i,name))
marks.sort()
def phase(ln):
    n='head'
    for i,name in marks:
        if ln>=i: n=name
    return n
fn=None; cur=None; agg=collections.defaultdict(collections.Counter)
for r in rows:
    if not r: continue
    if r[0]=="Function Name": fn=r[1][:50]; continue
    if r[0]=="File Path": cur=r[1].split("/")[-1]; continue
    try: ln,smp,inst=int(r[0]),int(r[4]),int(r[7])
    except: continue
    key=phase(ln) if cur=="pf_multicrop.cu" else "other:"+cur
    agg[fn][key+"|s"]+=smp; agg[fn][key+"|i"]+=inst
for fn,c in agg.items():
    ts=sum(v for k,v in c.items() if k.endswith("|s")) or 1; ti=sum(v for k,v in c.items() if k.endswith("|i")) or 1
    print(fn, "samples",ts,"inst",ti)
    keys=sorted({k[:-2] for k in c}, key=lambda k:-c[k+"|i"])
    for k in keys:
        if c[k+'|i'] or c[k+'|s']: print(f"   {k:22s} inst {100*c[k+'|i']/ti:5.1f}%  samples {100*c[k+'|s']/ts:5.1f}%")
