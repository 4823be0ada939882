import sys; sys.path.insert(0, '.')
from paper_2506_12718_b200 import bench_ops
for lg in (16, 18, 20, 22, 24):
    n = 1 << lg
    b = max(1, (1 << 24) // n)
    p = bench_ops.run("permute", 4, [n], b, reps=5)
    f = bench_ops.run("fft", 4, [n], b, reps=5)
    s = bench_ops.run("conv-std", 4, [n], b, reps=5)
    a = bench_ops.run("conv-pa", 4, [n], b, reps=5)
    print(lg, b, "share", round(p["median_s"] / f["median_s"], 3), "std/pa", round(s["median_s"] / a["median_s"], 3))
    b = 1
    p = bench_ops.run("permute", 4, [n], b, reps=5)
    f = bench_ops.run("fft", 4, [n], b, reps=5)
    s = bench_ops.run("conv-std", 4, [n], b, reps=5)
    a = bench_ops.run("conv-pa", 4, [n], b, reps=5)
    print(lg, b, "share", round(p["median_s"] / f["median_s"], 3), "std/pa", round(s["median_s"] / a["median_s"], 3))
