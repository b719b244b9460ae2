"""Run BASELINE configs 1, 3 and the 13 config-5 variants once each through
winograd_layer_conv with resident tensors (profiling driver for an ncu launch list)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2007_12216_b200 as rnsw
from paper_2007_12216_b200 import workloads as W

cases = []
c1, w1, x1 = W.config1()
cases.append((c1, w1, x1))
c3, w3, x3 = W.config3()
cases.append((c3, w3, x3))
w5, x5 = W.config5_operands()
for c5 in W.config5_cases():
    cases.append((c5, w5, x5))
for case, w, x in cases:
    spec = rnsw.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch,
                          tile_m=case.tile_m)
    system = rnsw.RnsSystem(case.moduli)
    bank = rnsw.precompute_filter_transforms(w, rnsw.reduce_for_system(rnsw.cached_transforms(case.tile_m, case.r), system))
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    for _ in range(2):
        rnsw.winograd_layer_conv(spec, wd, xd, system, declared_bound=case.declared_bound, filters=bank)
    torch.cuda.synchronize()
    print(case.name, flush=True)
