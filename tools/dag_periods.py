import numpy as np, sys
z=np.load(sys.argv[1]); tr=z['trace'].astype(np.int64); wk=z['walker'].astype(np.int64)
t0=tr[:,0].min(); w=(wk-t0)/1e3
n=len(w); per=np.diff(w[:,0])
print("steps",n,"end",w[-1,5] if w[-1,5]>0 else w[-1,3])
for a in range(0,n-1,10):
    b=min(a+10,n-1); seg=w[a:b]
    print("k %3d-%3d period %5.1f | wait %4.1f upd %4.1f diag %4.1f store+waitpanel %4.1f LU %4.1f"%(a,b,per[a:b].mean(),(seg[:,1]-seg[:,0]).mean(),(seg[:,2]-seg[:,1]).mean(),(seg[:,3]-seg[:,2]).mean(),(seg[:,4]-seg[:,3]).mean(),(seg[:,5]-seg[:,4]).mean()))
