import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_09582_b200 as glu
from paper_2307_09582_b200 import workloads
img = torch.from_numpy(workloads.scene(3840, 2160, 3, 0)).cuda()
low, grid = glu.grid_downsample(img, 8)
ctx = glu.glu.context()
c0 = ctx.close_sets
glu.optimize_field(img, low, grid, glu.GluConfig(), glu.Mode.Exact)
torch.cuda.synchronize()
n = ctx.close_sets - c0
print("recheck+close count", n, "fraction", n / (3840 * 2160))
