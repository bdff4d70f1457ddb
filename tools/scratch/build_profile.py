"""Phase timing of the config-4 variable-E d=10 system build: assembly,
concat_blocks, apply_dirichlet (synchronising timers)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07778_b200 import configs
tm = {}
t = time.perf_counter()
gsys, eps = configs.build_system(int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 10, tm)
torch.cuda.synchronize()
print("build", round(time.perf_counter() - t, 3), tm, "K ranks", max(gsys.K.ranks), flush=True)
