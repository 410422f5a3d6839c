import cProfile, pstats, sys
sys.path[:0] = ['.', 'tests']
import torch, cases as C, paper_1908_01906_b200 as B
from paper_1908_01906_b200 import device as DV
sc = C.build_scene(B, "radial59"); par = C.params(B, "radial59")
dev = DV.device_scene_for(sc)
for _ in range(20): DV.Epoch(dev, sc.meta_state(), par)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(500): DV.Epoch(dev, sc.meta_state(), par)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
