import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28706_b200 import problem as pb
from paper_2603_28706_b200.smoother import VankaLevel
from paper_2603_28706_b200.synth import CONFIGS, make_slab_inputs
cfg = CONFIGS["cfg1"]
syn = make_slab_inputs(cfg)
ctx = pb.make_context(cfg.nx, cfg.ny, cfg.k, pb.ModelParams(cfg.p, cfg.delta, cfg.nu, cfg.nu_inf), cfg.tau,
                      config=pb.DiscretizationConfig(40, 40, 1), v_minus=syn.v_minus)
lvl = VankaLevel(ctx, syn.U, pb.modified_newton(1.0), surrogate=(sys.argv[1] == "1"), rep_fraction=1.0)
print("built")
