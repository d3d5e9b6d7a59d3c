import sys
sys.path.insert(0, "/root/repo")
import faulthandler; faulthandler.enable()
import numpy as np
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200 import configs, _abi
_abi.check(_abi.lib().ibmi_tune(7, 16))
cfg = configs.get_config("c1")
a = configs.make_matrix("c1")
rep = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol, max_iterations=cfg.max_iterations, initial_guess="jacobi"))
print("ok", rep.iterations, rep.converged)
