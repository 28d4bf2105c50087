"""Wall time of sdd.quality_report (K5, host buffers in and out) on 513^2 and
1025^2 meshes: python tools/quality_time.py"""
import sys, numpy as np
sys.path.insert(0,'.')
from paper_1310_3435_b200 import sdd
ctx=sdd.Context(0)
U=sdd.RectDomain(0,1,0,1)
for n in (513,1025):
    x,y=np.meshgrid(np.linspace(0,1,n),np.linspace(0,1,n))
    X=x+0.05*np.sin(2*np.pi*x)*np.sin(np.pi*y); Y=y+0.05*np.sin(np.pi*x)*np.sin(2*np.pi*y)
    mesh=sdd.PhysicalMesh(n,n,U,X.ravel(),Y.ravel())
    import time
    for _ in range(3):
        t0=time.perf_counter(); q=sdd.quality_report(mesh,mesh,sdd.MonitorFunction.ring(),ctx=ctx); ms=(time.perf_counter()-t0)*1e3
    print(n, "quality_report wall ms (host buffers in and out)", round(ms,3), q.q_mean)
