import numpy as np, sys
a=np.fromfile(sys.argv[1],dtype=np.uint64).reshape(-1,3)
t0=a[:,0].astype(np.int64); t1=a[:,1].astype(np.int64); sm=(a[:,2]>>np.uint64(32)).astype(int); ns=(a[:,2]&np.uint64(0xffffffff)).astype(int)
T0=t0.min(); t0-=T0; t1-=T0
print("tiles",len(a),"kernel span us",t1.max()/1e3)
life=(t1-t0)/1e3
print("CTA life us: mean %.2f median %.2f p10 %.2f p90 %.2f max %.2f"%(life.mean(),np.median(life),np.percentile(life,10),np.percentile(life,90),life.max()))
# first wave = CTAs starting within first 1 us
fw=t0<1000
print("first-wave CTAs",fw.sum(),"life mean %.2f"%life[fw].mean(), " steady (start 20-80us) life mean %.2f"%life[(t0>20000)&(t0<80000)].mean())
# concurrency over time
edges=np.arange(0,t1.max()+1000,1000)
for e in edges[::4]:
    act=((t0<=e)&(t1>e)).sum()
    done=(t1<=e).sum()
    print("t=%5.1f us active %5d done %6d"%(e/1e3,act,done))
# throughput per 10us window in slots
for lo in range(0,int(t1.max()/1e3)+1,10):
    m=(t1/1e3>=lo)&(t1/1e3<lo+10)
    print("window %3d-%3d us: tiles finished %5d slots %7d"%(lo,lo+10,m.sum(),ns[m].sum()))
last=np.sort(t1)[-1332:]
print("last 1332 CTAs end between %.1f and %.1f us"%(last.min()/1e3,last.max()/1e3))
print("last start %.1f us"%(t0.max()/1e3))
