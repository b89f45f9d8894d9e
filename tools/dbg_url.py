import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, synth, oracle
from paper_1709_01190_b200 import flash
rp,col=synth.generate(synth.SHAPES['url'].with_(N=8000))
K,L,R,rng,seed,k=4,128,32,1<<15,0x5EED0002,128
o_ids,o_cnt=oracle.knn_graph(K,L,R,rng,seed,rp,col,k)
d_rp,d_col=flash.to_device_csr(rp,col)
with flash.FlashIndex(K,L,R,rng,seed) as idx:
    g_ids,g_cnt=idx.knn_graph(d_rp,d_col,k)
    a=flash.as_u32(idx.hash(d_rp,d_col,codes=False)[1])
g_ids=flash.as_u32(g_ids); g_cnt=flash.as_u32(g_cnt)
bad=np.where((g_ids!=o_ids).any(1)|(g_cnt!=o_cnt).any(1))[0]
print('bad rows',len(bad))
T=oracle.build(L,R,rng,seed,a,np.arange(8000,dtype=np.uint32))
sz=np.diff(T.off.astype(np.int64),axis=1)
M=np.array([sum(sz[t][a[q,t]] for t in range(L) if a[q,t]!=0xFFFFFFFF) for q in range(8000)])
print('M of bad', M[bad[:20]], 'M max', M.max())
for q in bad[:3]:
    j=np.where((g_ids[q]!=o_ids[q])|(g_cnt[q]!=o_cnt[q]))[0][0]
    print(q, j, 'gpu', list(zip(g_ids[q][j-2:j+4],g_cnt[q][j-2:j+4])), 'orc', list(zip(o_ids[q][j-2:j+4],o_cnt[q][j-2:j+4])))
for q in bad[:2]:
    print('q',q,'gpu',list(zip(g_ids[q][:6],g_cnt[q][:6])),'...',list(zip(g_ids[q][-4:],g_cnt[q][-4:])))
    print('q',q,'orc',list(zip(o_ids[q][:6],o_cnt[q][:6])),'...',list(zip(o_ids[q][-4:],o_cnt[q][-4:])))
    print('hist orc', np.bincount(o_cnt[q]), 'gpu', np.bincount(g_cnt[q]))
