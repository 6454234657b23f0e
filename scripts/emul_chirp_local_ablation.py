"""Accuracy diagnostic for the complex64 config-4 path: see the file body."""
import numpy as np, sys, math
src=open(__import__('os').path.join(__import__('os').path.dirname(__import__('os').path.abspath(__file__)), 'emul_chirp_local.py')).read()
# parametrise rounding of adds and multiplies
src=src.replace("def add(a,b): return Cx(a.x+b.x,a.y+b.y)\ndef sub(a,b): return Cx(a.x-b.x,a.y-b.y)",
"""MODE={'add':32,'mul':32}
def RA(v): return v if MODE['add']==64 else v.astype(np.float32)
def add(a,b):
    r=Cx.__new__(Cx); r.x=RA(a.x.astype(np.float64)+b.x); r.y=RA(a.y.astype(np.float64)+b.y); return r
def sub(a,b):
    r=Cx.__new__(Cx); r.x=RA(a.x.astype(np.float64)-b.x); r.y=RA(a.y.astype(np.float64)-b.y); return r""")
src=src.replace("class Cx:\n    __slots__=(\"x\",\"y\")\n    def __init__(s,x,y): s.x=r32(np.asarray(x)); s.y=r32(np.asarray(y))",
"""class Cx:
    __slots__=("x","y")
    def __init__(s,x,y):
        s.x=np.asarray(x); s.y=np.asarray(y)
        if MODE['mul']==32: s.x=r32(s.x); s.y=r32(s.y)""")
src=src.replace("def fma(a,b,c): return r32(a.astype(np.float64)*b.astype(np.float64)+c.astype(np.float64))",
"def fma(a,b,c):\n    v=np.asarray(a,np.float64)*np.asarray(b,np.float64)+np.asarray(c,np.float64)\n    return v if MODE['mul']==64 else r32(v)")
src=src.replace("    return Cx(fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,a.y*b.x))",
"    if MODE['mul']==64: return Cx(a.x.astype(np.float64)*b.x-a.y.astype(np.float64)*b.y, a.x.astype(np.float64)*b.y+a.y.astype(np.float64)*b.x)\n    return Cx(fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,a.y*b.x))")
src=src.replace("w=WORKLOADS[\"4\"]\nfor i in","w=WORKLOADS[\"4\"]\nfor i in []:#")
exec(src)
d=np.load('gpurun_out/diag_signals.npz')
for mode in [(32,32),(64,32),(32,64)]:
    MODE['add'],MODE['mul']=mode
    out=[]
    for j in range(len(d['idx'])):
        x=d['x'][j]; ref=d['ref'][j]
        X=kernel(x)
        out.append((np.abs(X-ref).max()/np.abs(ref).max(), np.linalg.norm(X-ref)/np.linalg.norm(ref)))
    print("add",mode[0],"mul",mode[1]," max-rel per signal", [f"{a:.2e}" for a,b in out], " rms-rel", [f"{b:.2e}" for a,b in out])
