"""Run the bench's C3 Gaussian-head step a few times (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(bench._bench_gauss_c3(torch.device("cuda", 0), 0, steps=3, cpu=False))
