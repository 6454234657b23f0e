"""Accuracy diagnostic for the complex64 config-4 path: see the file body."""
import numpy as np, scipy.fft as sf, sys, os
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2403_16665_b200.signals import WORKLOADS, generate
from concurrent.futures import ProcessPoolExecutor
w=WORKLOADS["4"]; N=M=8192; P=16384; L=8*N
k=np.arange(N); ph=(k.astype(np.int64)**2)%(2*L); c=np.exp(-1j*np.pi*ph/L)
h=np.zeros(P,complex); h[:M]=np.conj(c[:M]); h[P-N+1:]=np.conj(c[1:N][::-1])
H=np.fft.fft(h)/P; c64=c.astype(np.complex64); H64=H.astype(np.complex64)
def work(lo):
    B=512
    x=generate(w,lo,B,threads=1).astype(np.complex64)
    y=np.zeros((B,P),np.complex64); y[:,:N]=x*c64
    Y=sf.fft(y,axis=1,workers=1); Z=(Y*H64).astype(np.complex64)
    z=sf.ifft(Z,axis=1,workers=1)*np.float32(P)
    X32=z[:,:M]*c64
    yd=np.zeros((B,P),complex); yd[:,:N]=x.astype(complex)*c
    ref=np.fft.ifft(np.fft.fft(yd,axis=1)*H,axis=1)[:,:M]*P*c
    return (np.abs(X32-ref).max(axis=1)/np.abs(ref).max(axis=1))
n=int(sys.argv[1])
with ProcessPoolExecutor(8) as ex:
    e=np.concatenate(list(ex.map(work,range(0,n,512))))
print("scipy f32 chirp over",n,"max",e.max(),"p99.9",np.quantile(e,0.999),"median",np.median(e),"argmax",e.argmax())
