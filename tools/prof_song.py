import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2509_15948_b200.scheduler import execute_batched
from paper_2509_15948_b200.songs import desk_specs, search_song
dev = torch.device("cuda", 0)
def render(g, p, s):
    y, _ = execute_batched(g, p, s, device=dev); return y.cpu().numpy()
specs = desk_specs(3, seed=0)
inp = {i: bench.make_inputs(1000 + i, specs[i].tracks, specs[i].subgroups, specs[i].length, render) for i in range(3)}
search_song(specs[2], *inp[2], device=dev)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for i in range(2):
    search_song(specs[i], *inp[i], device=dev)
pr.disable()
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(25)
