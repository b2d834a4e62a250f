"""Prints the z-GEMM conditioning bound max_e B_e (ndg_tc_records) of seeded synthetic mixtures, the
quantities HotPath compares with TC_FORWARD_MAX_BOUND (RMS) and TC_FORWARD_PEAK_BOUND (max). Tuning aid."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2405_20067_b200 as ndg
from paper_2405_20067_b200 import datasets as D
for n, G, s0 in ((10, 100000, None), (10, 400, 0.3), (10, 400, None), (1, 273, None), (1, 50, None), (6, 4096, None), (16, 500000, None), (10, 1000, 0.02), (10, 1000, 0.05)):
    mix_np, sig = D.synthetic_mixture(n, G, seed=0, sigma0=s0)
    mix = ndg.Mixture.from_arrays(n, 0, **mix_np)
    hp = ndg.HotPath(n)
    r = hp.activate(mix)
    print(n, G, s0, round(float(sig), 4), "rms", round(r.tc_conditioning(), 1), "max", round(r.tc_cond_host[0], 1))
