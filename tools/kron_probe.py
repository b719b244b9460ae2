import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle
import paper_2007_12216_b200 as rnsw
SYS16 = (4001, 4331)
def run(b, h, c, k, tm, seed=0):
    rng = np.random.default_rng(seed)
    wt = np.clip(np.rint(rng.normal(0, 20, (3, 3, c, k))), -127, 127).astype(np.int8)
    x = rng.integers(0, 128, (b, h, h, c)).astype(np.int8)
    spec = rnsw.LayerSpec(h=h, w=h, c=c, k=k, r=3, padding=1, batch=b, tile_m=tm)
    system = rnsw.RnsSystem(SYS16)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    want = oracle.direct_conv_c(x, wt, 1)
    bad = np.argwhere(got != want)
    return len(bad), bad[:3].tolist()
for (b, h, c, k, tm) in [(32,28,256,256,8),(32,28,64,256,8),(32,28,256,64,8),(8,28,256,256,8),(1,28,256,256,8),(32,28,256,256,6),(32,28,256,256,10),(32,28,128,128,8),(9,28,64,64,8),(8,28,64,64,8),(16,28,32,64,8)]:
    print((b,h,c,k,tm), run(b,h,c,k,tm), flush=True)
