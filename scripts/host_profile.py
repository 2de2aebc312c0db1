"""cProfile of the bench's timed train steps (host-side cost per step)."""
import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_23044_b200 import trainer
WARM, STEPS = 3, 20
pr = cProfile.Profile()
orig = trainer.train_step
n = [0]
wall = []


def wrapped(*a, **k):
    n[0] += 1
    on = n[0] > WARM
    if on:
        pr.enable()
    t0 = time.perf_counter()
    r = orig(*a, **k)
    wall.append(time.perf_counter() - t0)
    if on:
        pr.disable()
    return r


trainer.train_step = wrapped
sys.argv = ["bench.py", "--steps", str(STEPS), "--warmup", str(WARM), "--cpu-tiles", "0"]
bench.main()
print("host wall per step ms:", [round(w * 1e3, 1) for w in wall])
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
