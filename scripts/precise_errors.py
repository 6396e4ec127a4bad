"""Measured errors of the reference-precision mode (precise.py) vs the float64 oracle, per sub-module
and per block, next to the bf16 product path's block error (profiles/r02_precise_errors.txt)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import evoformer_np as O
from paper_2203_00854_b200 import precise as PR, evoformer_block
from paper_2203_00854_b200.config import EvoConfig, init_block_params, synthetic_inputs

rel = lambda a, b: float(np.linalg.norm(np.asarray(a.double().cpu() if hasattr(a, "cpu") else a) - b) / np.linalg.norm(b))
for name, cfg in (("c32", EvoConfig(16, 32, 64, 32, 2, 1, 16)), ("c8", EvoConfig(16, 32, 64, 32, 8, 4, 16)),
                  ("ref", EvoConfig(8, 8, 16, 16, 2, 2, 8)), ("mid", EvoConfig(32, 64, 128, 64, 4, 2, 32))):
    for seed in (7, 31, 101):
        p = init_block_params(cfg, seed)
        m, z = synthetic_inputs(cfg, seed)
        rm, rz = O.evoformer_block(m, z, p, cfg)
        mo, zo = PR.evoformer_block(m, z, p, cfg)
        maxabs = max(float(np.abs(mo.double().cpu().numpy() - rm).max()), float(np.abs(zo.double().cpu().numpy() - rz).max()))
        bm, bz = evoformer_block(m, z, p, cfg)
        print(f"{name:4s} seed {seed:3d}: precise block rel m {rel(mo, rm):.2e} z {rel(zo, rz):.2e} max-abs {maxabs:.2e} "
              f"| bf16 product path rel m {rel(bm, rm):.2e} z {rel(bz, rz):.2e}")
