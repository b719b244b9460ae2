"""Per-config timings on one B200: BASELINE configs 1, 3 and the config-5
tile/residue sweep, each RNS-Winograd variant next to the direct int8
implicit-GEMM conv (tcgen05) on the same inputs.  Filters are precomputed
outside the timed region (rw/cli.py:459-463).  CUDA events, warm-up 3,
median of 10; every output is checked bit-exact against the direct conv.

usage: python tools/bench_configs.py [out.json]
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_12216_b200 as rnsw  # noqa: E402
from paper_2007_12216_b200 import workloads as W  # noqa: E402


def timed(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def run_case(case, w, x, direct_ref, xd, wd):
    spec = rnsw.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch,
                          tile_m=case.tile_m)
    system = rnsw.RnsSystem(case.moduli)
    bank = rnsw.precompute_filter_transforms(wd, rnsw.reduce_for_system(rnsw.cached_transforms(case.tile_m, case.r),
                                                                       system))
    run = lambda: rnsw.winograd_layer_conv(spec, wd, xd, system, declared_bound=case.declared_bound, filters=bank)
    y = run()
    exact = bool(torch.equal(y, direct_ref))
    ms = timed(run)
    st = rnsw.StageTimings()
    for _ in range(3):
        rnsw.winograd_layer_conv(spec, wd, xd, system, declared_bound=case.declared_bound, filters=bank, timings=st)
    return dict(name=case.name, tile=f"F({case.tile_m}x{case.tile_m},{case.r}x{case.r})", n=case.tile_m + case.r - 1,
                moduli=list(case.moduli), ms=round(ms, 4), tops=round(case.direct_ops() / ms / 1e9, 2),
                exact=exact, stages_ms={k: round(v / 3 * 1e3, 4) for k, v in
                                        (("input_transform", st.input_transform), ("gemm", st.gemm),
                                         ("output_transform", st.backward_transform))})


def main():
    out = {"device": torch.cuda.get_device_name(), "cases": []}
    for label, (case, w, x) in (("config1", W.config1()), ("config3", W.config3())):
        wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
        spec = rnsw.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch)
        packed = rnsw.DirectWeights(wd)
        direct = rnsw.direct_conv(spec, wd, xd, packed)
        dms = timed(lambda: rnsw.direct_conv(spec, wd, xd, packed))
        res = run_case(case, w, x, direct, xd, wd)
        res.update(config=label, direct_ms=round(dms, 4), direct_tops=round(case.direct_ops() / dms / 1e9, 2))
        out["cases"].append(res)
        print(json.dumps(res), flush=True)
    w, x = W.config5_operands()
    wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
    spec = rnsw.LayerSpec(h=28, w=28, c=256, k=256, r=3, padding=1, batch=32)
    packed = rnsw.DirectWeights(wd)
    direct = rnsw.direct_conv(spec, wd, xd, packed)
    dms = timed(lambda: rnsw.direct_conv(spec, wd, xd, packed))
    ops = W.config5_cases()[0].direct_ops()
    out["config5_direct"] = dict(ms=round(dms, 4), tops=round(ops / dms / 1e9, 2))
    print(json.dumps(out["config5_direct"]), flush=True)
    for case in W.config5_cases():
        res = run_case(case, w, x, direct, xd, wd)
        res.update(config="config5", direct_ms=round(dms, 4), direct_tops=out["config5_direct"]["tops"])
        out["cases"].append(res)
        print(json.dumps(res), flush=True)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
