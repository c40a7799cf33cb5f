import sys; sys.path.insert(0, '/root/repo')
import paper_2004_02583_b200 as tk
ctx = tk.Context(0)
for n in (655360, 33554432, 400000000):
    ctx.uniform01(7, 1, n)
