"""Split an ncu source-page CSV (ncu -i rep --page source --csv) into contiguous SASS regions of similar
execution count and print, per region, its share of the stall samples and of the executed instructions with
the leading stall reasons: python tools/ncu_regions.py source.csv"""
import csv,sys
r=csv.reader(open(sys.argv[1]))
next(r); h=next(r)
ix={n:i for i,n in enumerate(h)}
rows=[row for row in r if len(row)==len(h)]
tot=sum(int(x[ix['# Samples']]) for x in rows)
exe=sum(int(x[ix['Instructions Executed']]) for x in rows)
def E(x): return int(x[ix['Instructions Executed']])
def S(x): return int(x[ix['# Samples']])
print('instr',len(rows),'samples',tot,'exec %.1fG'%(exe/1e9))
# contiguous regions by similar exec counts
regs=[];start=0
import math
def cls(e):
    return 0 if e==0 else int(math.log(e,1.6))
for i in range(1,len(rows)+1):
    if i==len(rows) or cls(E(rows[i]))!=cls(E(rows[start])):
        regs.append((start,i)); start=i
# merge tiny regions? just print those with samples > 0.5%
keys=['stall_wait','stall_selected','stall_no_inst','stall_branch_resolving','stall_dispatch','stall_short_sb','stall_math','stall_barrier','stall_long_sb']
for a,b in regs:
    s=sum(S(x) for x in rows[a:b])
    if s/tot>0.004:
        e=sum(E(x) for x in rows[a:b])
        d={k:sum(int(x[ix[k]]) for x in rows[a:b]) for k in keys}
        print(a,b,'n=%d'%(b-a),'exec/instr=%.3g'%(E(rows[a])),'samples=%.1f%%'%(100*s/tot),'exec=%.1f%%'%(100*e/exe),' '.join('%s=%.1f'%(k[6:],100*v/tot) for k,v in d.items() if v/tot>0.002))
