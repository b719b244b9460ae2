"""Run the fused VGG16 stack once at batch B (default 256) without a CUDA
graph: the driver for the per-launch ncu list (times + DRAM traffic)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2007_12216_b200 import workloads as W
from paper_2007_12216_b200.vgg import VGG16Rns

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
net = VGG16Rns()
x = torch.from_numpy(W.vgg16_images(B)).cuda()
net.forward_fused(x)
torch.cuda.synchronize()
print("ok", B)
