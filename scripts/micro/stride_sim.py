#!/usr/bin/env python3
"""Bank-conflict simulation of the rectangle's priv-row gathers (kernels.cuh rect_run)
for each priv row stride mod 32 on seeded C3 columns: lanes own target pairs
(t, t + 16), half-warps the bottoms of a pair; a gather costs the largest number of
distinct words in one bank.  usage: stride_sim.py [stride mod 32 ...]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from inputs import synth
from oracle import oracle as orc
W,H,S,D=1024,440,5,128
imgs=[synth.frame(3,i,W,H,D) for i in range(3)]
cols=np.concatenate([orc.reduce(im,S,4,0xFFFF,D) for im in imgs])  # [n][H], -1? invalid marker
print(cols.shape, cols.min(), cols.max())
def fmat(col):
    valid = (col>=0)&(col < (D<<8))
    dO=np.minimum(col, ((D-1)<<8)+127)
    t=np.where(valid, dO+128, 0).astype(np.int64); n=valid.astype(np.int64)
    T=np.concatenate([[0],np.cumsum(t)]); N=np.concatenate([[0],np.cumsum(n)])
    return T,N
strides=[int(x) for x in sys.argv[1:]] or [1,3,15,17,19,5,9,13]
res={s:[0,0] for s in strides}
rng=np.random.default_rng(0)
for ci in rng.choice(len(cols), 60, replace=False):
    T,N=fmat(cols[ci])
    nb=(H+31)//32
    for b in range(nb-1):
        Kn=32*(b+1)
        for jA in range(1, 32*(b+1), 2):  # bottoms j final up to block b... all bottoms <= Kn
            for tt in (0,16):
                addrs=[]
                for lane in range(32):
                    t=(lane&15)+tt; hw=lane>>4; j=jA+hw
                    k=min(Kn+t,H-1)
                    if j>k: j=k
                    n=N[k+1]-N[j]
                    f=0 if n==0 else int(((T[k+1]-T[j])//128)//(2*n))
                    addrs.append((k-Kn, f))
                for s in strides:
                    banks={}
                    for (r,f) in set(addrs):
                        bk=(r*s+f)%32
                        banks[bk]=banks.get(bk,0)+1
                    res[s][0]+=max(banks.values()); res[s][1]+=1
for s in strides: print('stride %% 32 = %2d: %.3f wf per gather'%(s,res[s][0]/res[s][1]))
