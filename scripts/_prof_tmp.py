import sys,collections
import numpy as np
d=collections.defaultdict(lambda: np.zeros(4)); rows={}
for l in open(sys.argv[1]):
    if l.startswith("PROF"):
        f=l.split()[1:]; c=int(f[0]); d[c]+=np.array([float(x) for x in f[1:5]]); rows[c]=int(f[5])
cs=sorted(d)
w=np.array([d[c][1]/d[c][0]/1.965e3 for c in cs]); b=np.array([d[c][2]/d[c][0]/1.965e3 for c in cs]); sp=np.array([d[c][3]/d[c][0]/1.965e3 for c in cs])
print("work us: mean %.3f min %.3f max %.3f; barrier mean %.3f min %.3f max %.3f; spmv mean %.3f max %.3f"%(w.mean(),w.min(),w.max(),b.mean(),b.min(),b.max(),sp.mean(),sp.max()))
for c in cs: print(c, rows[c], "%.3f %.3f %.3f"%(d[c][1]/d[c][0]/1.965e3, d[c][2]/d[c][0]/1.965e3, d[c][3]/d[c][0]/1.965e3))
