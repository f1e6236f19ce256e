"""SASS instruction mix of an attention ncu report (--page source), per 32 exps at the c4 SP=8 shape
(N = 75600, H = 5): python tools/ncu_inst_mix.py REPORT.ncu-rep.  Development aid."""
import csv,collections,subprocess,sys
f=sys.argv[1]
out=subprocess.run(['ncu','-i',f,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
h=rows[1]; R=rows[2:]
ia=h.index("Instructions Executed"); isrc=h.index("Source"); ismp=h.index("Warp Stall Sampling (All Samples)")
tot=collections.Counter(); smp=collections.Counter()
for r in R:
    op=r[isrc].split()
    if not op: continue
    o=op[0]
    if o.startswith('@'): o=op[1]
    o=o.split('.')[0] if not o.startswith('UTC') else o
    tot[o]+=int(r[ia] or 0); smp[o]+=int(r[ismp] or 0)
E=75600*75600*5/32
S=sum(smp.values())
print(f, "warp-inst per 32 exps:", round(sum(tot.values())/E,2))
for o,n in tot.most_common(22): print(f"  {o:14s} {n/E:6.3f}  samples {smp[o]/S*100:5.1f}%")
