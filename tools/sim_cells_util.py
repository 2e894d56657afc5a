#!/usr/bin/env python
"""CPU estimate (numpy, synthetic clouds only) of the lane utilisation alternative CELLS accept
schemes would reach on C3 / C5, used to decide against them:

  * "(c,k)-uniform": the warp walks (centre, point-of-lane) combinations and the lanes whose
    pair passed the filter decide in place (no compaction) -- utilisation = candidates per
    32-point chunk with any candidate / 32;
  * private per-lane queues with lane = centre -- utilisation = mean / max candidates per
    centre within a 128-point warp tile;
  * how many (8-centre batch x 128-point tile) combinations hold no candidate at all (what a
    perfect spatial cull of the filter could skip), and how often a tile / half tile
    overflows the 960-entry ring.

  python tools/sim_cells_util.py 3      # config 3;   ... 5 [W]

The visited set here is the group's bounding box (no per-row hulls), so the pass rate is lower
than the engine's (0.17 vs 0.22 on C3).
"""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import clouds
cfg_id=int(sys.argv[1]); 
cfg=clouds.CONFIGS[cfg_id]
Wd=int(sys.argv[2]) if len(sys.argv)>2 else cfg['W']
P,Nn=clouds.make_cloud(cfg_id); P=P.astype(np.float64); Nn=Nn.astype(np.float64)
C=clouds.make_centres(cfg_id,len(P))
W=Wd; b=cfg['b']; cosA=cfg['cos_As']
R=np.sqrt((W*b)**2+(W*b/2+b)**2)
h=R/8
lo=P.min(0); 
cell=np.floor((P-lo)/h).astype(np.int64)
dim=cell.max(0)+1
key=(cell[:,2]*dim[1]+cell[:,1])*dim[0]+cell[:,0]
srt=np.argsort(key,kind='stable'); Ps=P[srt]; Ns=Nn[srt]; ks=key[srt]; cs=cell[srt]
# morton order of centres
def spread(v):
    v=v.astype(np.uint64)&0x3ff
    v=(v|(v<<16))&0x30000ff; v=(v|(v<<8))&0x300f00f; v=(v|(v<<4))&0x30c30c3; v=(v|(v<<2))&0x9249249
    return v
cp=P[C]; q=np.floor((cp-lo)/(P.max(0)-lo).max()*1023).astype(np.int64)
mk=spread(q[:,0])|(spread(q[:,1])<<1)|(spread(q[:,2])<<2)
corder=C[np.argsort(mk,kind='stable')]
rng=np.random.default_rng(0)
G=32
tot_pass=0; tot_vis=0; act_chunks=0; tot_chunks=0; lane_max_sum=0; lane_mean_sum=0
hist=np.zeros(33)
for gi in rng.choice(len(corder)//G, 60, replace=False):
    cen=corder[gi*G:(gi+1)*G]; cP=P[cen]; cN=Nn[cen]
    bl=np.floor((cP.min(0)-R-lo)/h).astype(int).clip(0); bh=np.floor((cP.max(0)+R-lo)/h).astype(int)
    m=np.all((cs>=bl)&(cs<=bh),axis=1)
    X=Ps[m]; NX=Ns[m]   # already in (z,y,x) cell order
    # row hull skipped (box)
    d=X[None,:,:]-cP[:,None,:]
    be=np.einsum('gpk,gk->gp',d,cN); dd=(d*d).sum(-1); al2=dd-be*be
    s=np.einsum('pk,gk->gp',NX,cN)
    u=W/2-be/b; w=al2/b/b
    ok=(s>=cosA)&(u>-1)&(u<=W-1)&(w<=(W-1)**2)
    insph=dd<=R*R
    n=X.shape[0]; nch=n//32
    okc=ok[:,:nch*32].reshape(G,nch,32)
    cnt=okc.sum(-1)  # per centre, chunk
    tot_pass+=cnt.sum(); tot_vis+=G*nch*32; act_chunks+=(cnt>0).sum(); tot_chunks+=G*nch
    hist+=np.bincount(cnt.ravel(),minlength=33)
    # private queue utilization: per warp tile of 128 points, lane=centre counts
    nt=n//128
    c128=ok[:,:nt*128].reshape(G,nt,128).sum(-1)  # centre, tile
    lane_max_sum+=c128.max(0).sum(); lane_mean_sum+=c128.mean(0).sum()
print('cfg',cfg_id,'W',W,'pass/visited',tot_pass/tot_vis,'U (c,k-uniform)=',tot_pass/(32*act_chunks),'active chunk frac',act_chunks/tot_chunks)
print('private-queue util per 128-tile (mean/max):',lane_mean_sum/lane_max_sum)
print('hist of per-(centre,32chunk) counts:',(hist/hist.sum()).round(3))
# batch-of-8 x warp tile emptiness
import itertools
emp_c=0; emp_s=0; tot=0; emp1=0; tot1=0; big=0; tiles=0
for gi in rng.choice(len(corder)//G, 40, replace=False):
    cen=corder[gi*G:(gi+1)*G]; cP=P[cen]; cN=Nn[cen]
    bl=np.floor((cP.min(0)-R-lo)/h).astype(int).clip(0); bh=np.floor((cP.max(0)+R-lo)/h).astype(int)
    m=np.all((cs>=bl)&(cs<=bh),axis=1)
    X=Ps[m]; NX=Ns[m]
    d=X[None,:,:]-cP[:,None,:]
    be=np.einsum('gpk,gk->gp',d,cN); dd=(d*d).sum(-1); al2=dd-be*be
    s=np.einsum('pk,gk->gp',NX,cN)
    u=W/2-be/b; w=al2/b/b
    ok=(s>=cosA)&(u>-1)&(u<=W-1)&(w<=(W-1)**2)
    n=X.shape[0]; nt=n//128
    okt=ok[:,:nt*128].reshape(4,8,nt,128).sum(-1).sum(1)   # batch, tile
    emp_c+=(okt==0).sum(); tot+=okt.size
    ok1=ok[:,:nt*128].reshape(G,nt,128).sum(-1)
    emp1+=(ok1==0).sum(); tot1+=ok1.size
    tt=ok1.sum(0); big+=(tt>960).sum(); tiles+=nt
    half=ok[:,:nt*128].reshape(2,16,nt,128).sum(-1).sum(1)
    bigh=(half>960).sum()
print('empty (8-centre batch x 128 contiguous tile):',emp_c/tot,' empty (centre x tile):',emp1/tot1)
print('tiles > 960 candidates:',big/tiles,' half-tiles > 960:',bigh/ (2*nt))
