import time, numpy as np
import paper_1611_01391_b200 as s
A = s.gen_factor_gaussian(256, 256, 8, 1e-8, s.Rng(0))
for _ in range(3):
    g = s.cross_approx(A, 8, 16, 16, [], 3, 1.1, s.Rng(1)); s.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
s.synchronize()
N = 50
t0 = time.perf_counter()
for _ in range(N): g = s.cross_approx(A, 8, 16, 16, [], 3, 1.1, s.Rng(1))
t1 = time.perf_counter()
for _ in range(N): s.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
t2 = time.perf_counter()
print("cross_approx %.3f ms, cur_evaluate %.3f ms" % ((t1 - t0) / N * 1e3, (t2 - t1) / N * 1e3))
s.set_timing(True)
g = s.cross_approx(A, 8, 16, 16, [], 3, 1.1, s.Rng(1)); s.cur_evaluate(A, g["I"], g["J"], g["nucleus"])
print(s.timing_report())
