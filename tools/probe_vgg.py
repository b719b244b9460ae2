"""Probe: per-layer, per-kernel device times of the VGG16 RNS stack, and a
bit-exact check of the batch-1 stack against the CPU oracle."""
import sys, time, json
from collections import defaultdict
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2007_12216_b200 import workloads as W
from paper_2007_12216_b200.vgg import VGG16Rns

batches = [int(b) for b in (sys.argv[1:] or ["1", "32"])]
net = VGG16Rns()
for B in batches:
    x = torch.from_numpy(W.vgg16_images(B)).cuda()
    for _ in range(2):
        net.forward(x)
    torch.cuda.synchronize()
    rec = []
    net.forward_staged(x, lambda kind, i, a, b: rec.append((kind, i, a, b)))
    torch.cuda.synchronize()
    per = defaultdict(float)
    rows = defaultdict(dict)
    for kind, i, a, b in rec:
        t = a.elapsed_time(b)
        per[kind] += t
        rows[i][kind] = t
    tot = sum(per.values())
    work = net.layer_work(B)
    print(f"B={B} total {tot:.3f} ms  " + "  ".join(f"{k} {v:.3f}" for k, v in per.items()))
    for i, r in rows.items():
        wk = work[i]
        mid = (f"  gemm {wk['gemm_ops']/r['gemm']/1e9:6.0f} TOPS" if "gemm" in r else
               f"  prod {wk['product_bytes']/r['product']/1e6:6.0f} GB/s")
        print(f"  {wk['name']:8s} " + " ".join(f"{k[:6]} {v:7.3f}" for k, v in r.items()) +
              f"  in {wk['input_transform_bytes']/r['input_transform']/1e6:6.0f} GB/s" + mid +
              f"  out {wk['output_transform_bytes']/r['output_transform']/1e6:6.0f} GB/s")
    print(f"  direct-equiv {sum(w['direct_ops'] for w in work)/tot/1e9:.1f} TOPS")
    for _ in range(2):  # warm-up: lazy module loading of the fused instances
        net.forward_fused_staged(x, lambda *a: None)
    torch.cuda.synchronize()
    rec = []
    net.forward_fused_staged(x, lambda kind, i, a, b: rec.append((kind, i, a, b)))
    torch.cuda.synchronize()
    perf = defaultdict(float)
    for kind, i, a, b in rec:
        perf[kind] += a.elapsed_time(b)
    totf = sum(perf.values())
    print(f"B={B} fused total {totf:.3f} ms  " + "  ".join(f"{k} {v:.3f}" for k, v in perf.items()) +
          f"  direct-equiv {sum(w['direct_ops'] for w in work)/totf/1e9:.1f} TOPS")
if "--check" in sys.argv or True:
    import oracle
    from oracle.vgg_ref import vgg16_stack
    x = W.vgg16_images(1)
    got, outs = net.forward(torch.from_numpy(x).cuda(), keep_int32=True)
    t = time.time()
    want, wouts = vgg16_stack(x, net.weights, W.VGG16_LAYERS, W.VGG16_SHIFTS, keep_int32=True)
    print("oracle stack", time.time() - t, "s")
    for i, (a, b) in enumerate(zip(outs, wouts)):
        assert np.array_equal(a.cpu().numpy(), b), f"layer {i} int32 mismatch"
    assert np.array_equal(got.cpu().numpy(), want)
    print("VGG16 b=1 bit-exact vs direct conv: all 13 layers")
