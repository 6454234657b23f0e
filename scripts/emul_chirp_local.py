"""Accuracy diagnostic for the complex64 config-4 path: see the file body."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2403_16665_b200.signals import WORKLOADS, generate
f32=np.float32
def r32(a): return a.astype(np.float32)
def fma(a,b,c): return r32(a.astype(np.float64)*b.astype(np.float64)+c.astype(np.float64))
class Cx:
    __slots__=("x","y")
    def __init__(s,x,y): s.x=r32(np.asarray(x)); s.y=r32(np.asarray(y))
def add(a,b): return Cx(a.x+b.x,a.y+b.y)
def sub(a,b): return Cx(a.x-b.x,a.y-b.y)
def cmul(a,b, mode=0):
    # FMUL + FFMA per component
    if mode==0: return Cx(fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,a.y*b.x))
    return Cx(fma(-a.y,b.y,a.x*b.x), fma(a.y,b.x,a.x*b.y))
def conj(a): return Cx(a.x,-a.y)
import math
def cospi16(k):
    return math.cos(k*math.pi/16)
def tw_const(xc,e,R):
    k=((32//R)*e)&31
    if k==0: return xc
    if k==16: return Cx(-xc.x,-xc.y)
    if k==8: return Cx(xc.y,-xc.x)
    if k==24: return Cx(-xc.y,xc.x)
    h=f32(0.70710678118654752440084436210485)
    if k==4: return Cx((xc.x+xc.y)*h,(xc.y-xc.x)*h)
    if k==12: return Cx((xc.y-xc.x)*h,-(xc.x+xc.y)*h)
    c=f32(math.cos(k*math.pi/16)); s=f32(math.sin(k*math.pi/16))
    return Cx(fma(xc.x,np.full_like(xc.x,c),xc.y*s), fma(xc.y,np.full_like(xc.y,c),-(xc.x*s)))
def bitrev(i,bits):
    r=0
    for b in range(bits): r|=((i>>b)&1)<<(bits-1-b)
    return r
def dft_reg(v):  # list of Cx length R
    R=len(v); half=R//2
    while half>=1:
        for base in range(0,R,2*half):
            for k in range(half):
                a=v[base+k]; b=v[base+k+half]
                v[base+k]=add(a,b); v[base+k+half]=tw_const(sub(a,b),k*(R//(2*half)),R)
        half//=2
    bits=int(math.log2(R))
    return [v[bitrev(i,bits)] for i in range(R)]
def exact(e,L):
    ang=2*np.pi*(np.asarray(e)%L)/L
    return Cx(np.cos(ang),-np.sin(ang))
N=M=8192; P=16384; L=8*N
k=np.arange(N)
ph=(k.astype(np.int64)**2)%(2*L); c=np.exp(-1j*np.pi*ph/L)
h=np.zeros(P,complex); h[:M]=np.conj(c[:M]); h[P-N+1:]=np.conj(c[1:N][::-1])
H=np.fft.fft(h)/P
def czt64(x):
    y=np.zeros(P,complex); y[:N]=x.astype(np.complex128)*c[:N]
    return (np.fft.ifft(np.fft.fft(y)*H)*P)[:M]*c[:M]
def kernel(x, twmode="exact"):
    n=np.arange(1024)
    cx=Cx(c.real,c.imag)
    xx=Cx(x.real,x.imag)
    # input v[i][n] = x[n+1024 i]*c ; i<8
    v=[]
    for i in range(16):
        if i<8:
            idx=n+1024*i
            v.append(cmul(Cx(xx.x[idx],xx.y[idx]),Cx(cx.x[idx],cx.y[idx])))
        else: v.append(Cx(np.zeros(1024),np.zeros(1024)))
    v=dft_reg(v)                      # P1 DIF over i -> k1
    v=[v[0]]+[cmul(v[r],exact(r*n,P)) for r in range(1,16)]   # twiddle W^{n k1}
    # y[k1][n]; P2 over n = n' + 256 i'
    Y=v
    out=[[None]*4 for _ in range(16)]   # z[k1][k2] arrays over n' (256)
    np_=np.arange(256)
    for k1 in range(16):
        a=[Cx(Y[k1].x[np_+256*i],Y[k1].y[np_+256*i]) for i in range(4)]
        a=dft_reg(a)
        for k2 in range(4):
            out[k1][k2]= a[k2] if k2==0 else cmul(a[k2],exact(np_*k2,1024))
    # P3: for each (k1,k2): n' = n'' + 16 i'' -> DFT16 over i''
    W=[[None]*4 for _ in range(16)]
    nn=np.arange(16)
    for k1 in range(16):
        for k2 in range(4):
            z=out[k1][k2]
            a=[Cx(z.x[nn+16*i],z.y[nn+16*i]) for i in range(16)]
            a=dft_reg(a)
            W[k1][k2]=[a[0]]+[cmul(a[k3],exact(nn*k3,256)) for k3 in range(1,16)]  # each over n'' (16)
    # P4: DFT16 over n'' for each (k1,k2,k3) -> k4
    Yf=np.zeros(P,np.complex64)
    Z={}
    Hc=H.astype(np.complex64)
    for k1 in range(16):
        for k2 in range(4):
            for k3 in range(16):
                w_=W[k1][k2][k3]
                a=[Cx(w_.x[i:i+1],w_.y[i:i+1]) for i in range(16)]
                a=dft_reg(a)
                for k4 in range(16):
                    f=k1+16*k2+64*k3+1024*k4
                    hv=Cx(np.array([Hc[f].real]),np.array([Hc[f].imag]))
                    Z[(k1,k2,k3,k4)]=conj(cmul(a[k4],hv))
    # Q1: DFT16 over k4 -> n''
    Wq=[[None]*4 for _ in range(16)]
    for k1 in range(16):
        for k2 in range(4):
            cols=[]
            for k3 in range(16):
                a=dft_reg([Z[(k1,k2,k3,k4)] for k4 in range(16)])   # index n''
                cols.append(a)
            # Q2: for each n'': twiddle W256^{n'' k3}, DFT16 over k3 -> i''
            zz=Cx(np.zeros(256),np.zeros(256))
            for n2 in range(16):
                a=[cols[k3][n2] for k3 in range(16)]
                a=[a[0]]+[cmul(a[k3],exact(np.array([n2*k3]),256)) for k3 in range(1,16)]
                a=dft_reg(a)
                for i2 in range(16):
                    zz.x[n2+16*i2]=a[i2].x[0]; zz.y[n2+16*i2]=a[i2].y[0]
            Wq[k1][k2]=zz
    # Q3: for each k1, n' <256: twiddle W1024^{n' k2}, DFT4 over k2 -> i'
    yq=[None]*16
    for k1 in range(16):
        a=[Wq[k1][k2] if k2==0 else cmul(Wq[k1][k2],exact(np_*k2,1024)) for k2 in range(4)]
        a=dft_reg(a)
        arr=Cx(np.zeros(1024),np.zeros(1024))
        for i in range(4):
            arr.x[np_+256*i]=a[i].x; arr.y[np_+256*i]=a[i].y
        yq[k1]=arr
    # Q4: twiddle W^{n k1}, DFT16 over k1 -> i; output n+1024 i
    a=[yq[0]]+[cmul(yq[k1],exact(n*k1,P)) for k1 in range(1,16)]
    a=dft_reg(a)
    X=np.zeros(M,complex)
    for i in range(8):
        o=cmul(conj(a[i]),Cx(cx.x[n+1024*i],cx.y[n+1024*i]))
        X[n+1024*i]=o.x.astype(np.float64)+1j*o.y.astype(np.float64)
    return X
w=WORKLOADS["4"]
for i in [int(a) for a in sys.argv[1:]]:
    x=generate(w,i,1,threads=1)[0].astype(np.complex64)
    ref=czt64(x)
    X=kernel(x)
    print(i, f"{np.abs(X-ref).max()/np.abs(ref).max():.3e}")

if __name__ == "__main__" and len(sys.argv) == 1:
    pass
