"""Per-layer latencies of BASELINE configs 1, 3, 5 (bench.py's layer_configs)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
r = bench.layer_config_latencies(torch)
print(json.dumps({k: (v["ms"], v["direct_tcgen05_ms"]) for k, v in r.items()}))
