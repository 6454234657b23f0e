"""Accuracy diagnostic for the complex64 config-4 path: see the file body."""
import numpy as np, scipy.fft as sf, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2403_16665_b200.signals import WORKLOADS, generate
from concurrent.futures import ProcessPoolExecutor
w=WORKLOADS["4"]; N=M=8192; r=8
n=np.arange(N)
def work(lo):
    B=256
    x=generate(w,lo,B,threads=1).astype(np.complex64)
    X=np.zeros((B,M),np.complex64); ref=np.zeros((B,M),complex)
    for c in range(r):
        tw=np.exp(-2j*np.pi*((c*n)%(r*N))/(r*N))
        y=(x*tw.astype(np.complex64)).astype(np.complex64)
        Y=sf.fft(y,axis=1,workers=1)
        X[:,c::r]=Y[:,:N//r]
        ref[:,c::r]=np.fft.fft(x.astype(complex)*tw,axis=1)[:,:N//r]
    return np.abs(X-ref).max(axis=1)/np.abs(ref).max(axis=1)
nb=int(sys.argv[1])
with ProcessPoolExecutor(8) as ex:
    e=np.concatenate(list(ex.map(work,range(0,nb,256))))
print("scipy f32 residue alpha-FFT over",nb,"max",e.max(),"p99.9",np.quantile(e,0.999),"median",np.median(e),"argmax",e.argmax())
