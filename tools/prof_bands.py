import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
import torch
import paper_2307_09582_b200 as glu
from paper_2307_09582_b200 import workloads, bands
img = torch.from_numpy(workloads.scene(7680, 4320, 5)).cuda()
for world in (2, 8):
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        r = bands.joint_optimize_banded_local(img, 16, world)
        torch.cuda.synchronize(); dt = time.time() - t
    print("world", world, "ms", dt * 1e3)
pr = cProfile.Profile(); pr.enable()
r = bands.joint_optimize_banded_local(img, 16, 8); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
