"""Time the input transform stage (rnsw_input_transform) on a VGG16 layer
shape: python tools/time_k1.py [layer] [batch] [reps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2007_12216_b200 import _native, workloads as W
from paper_2007_12216_b200.layer import plan_for, _stream_ptr
from paper_2007_12216_b200.residue import RnsSystem
from paper_2007_12216_b200.transforms import cached_transforms

name = sys.argv[1] if len(sys.argv) > 1 else "conv1_2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
_, side, c, k, _ = {l[0]: l for l in W.VGG16_LAYERS}[name]
plan = plan_for(cached_transforms(14, 3), RnsSystem((4001, 4331)))
l = _native.lib()
x = torch.randint(0, 128, (B, side, side, c), dtype=torch.int8, device="cuda")
tiles = B * ((side + 13) // 14) ** 2
vb = l.rnsw_v_bytes(plan.handle, tiles, c)
V = torch.empty(vb, dtype=torch.uint8, device="cuda")
vp = _native.c_void_p
call = lambda: _native.check(l.rnsw_input_transform(plan.handle, vp(x.data_ptr()), B, side, side, c, 1, 0,
                                                     vp(V.data_ptr()), vb, _stream_ptr()))
for _ in range(3):
    call()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); call(); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
ms = min(ts)
gb = (B * side * side * c + vb) / 1e9
print(f"{name} B={B}: {ms*1e3:.1f} us  {gb/ms*1e3:.0f} GB/s")
