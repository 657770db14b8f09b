"""Probe: does concurrent PCIe DMA (H2D / D2H on a side stream) slow the solve?
usage: python tools/dma_probe.py"""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
gc = load_case('/root/repo/cases/synth9241.m'); T = 10000; n = gc.n_bus
vm0, va0 = gc.v_start(); p0, q0 = montecarlo(gc, T)
plan = S.NrPlan.from_case(gc, device=0, profile=1); plan.stage(p0, q0, vm0, va0); plan.run()
h = torch.empty((n, T), dtype=torch.float64).pin_memory(); d = torch.empty((n, T), dtype=torch.float64, device='cuda')
side = torch.cuda.Stream()
for mode in ('none', 'h2d', 'd2h', 'both', 'none'):
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for _ in range(4):
            if mode in ('h2d', 'both'): d.copy_(h, non_blocking=True)
            if mode in ('d2h', 'both'): h.copy_(d, non_blocking=True)
    plan.run()
    tm = plan.timing()
    print(mode, f"total {tm['total_ms']:.2f} lu {tm['lu_ms']/max(tm['lu_launches'],1):.3f} npm {tm['npm_ms']/max(tm['npm_launches'],1):.3f} bs {tm['fsbs_ms']/max(tm['fsbs_launches'],1):.3f}", flush=True)
    torch.cuda.synchronize()
