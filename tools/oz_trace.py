import sys, os, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2502_06377_b200 import configs, _abi
from paper_2502_06377_b200.device import DeviceSolver
L = _abi.lib()
a = torch.as_tensor(configs.make_matrix("c4"), device="cuda")
cfg = configs.get_config("c4")
ds = DeviceSolver(a, partition=cfg.partition())
ds.set_emulation(16)
ds.setup(); ds.init_sigma(0)
ds.sweep(1e-9, 5000)
os.environ["IBMI_OZ_TRACE"] = "1"
print(ds.sweep_timed(1e-9, 5000)[3]); torch.cuda.synchronize()
