#!/usr/bin/env python3
"""Kernel timeline of one decomposition step (CUPTI through torch.profiler):
per-kernel start/end on the device, the busy fraction of the step and the
largest idle gaps with the kernels on either side. Used to find host-side
stalls between launches (the per-class kernel times in bench.py do not see
them).

usage: python tools/timeline.py --config 5 [--warm 2] [--gaps 15]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2004_02583_b200 as tk  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--warm", type=int, default=2)
    p.add_argument("--gaps", type=int, default=15)
    p.add_argument("--dump", action="store_true", help="print every activity (start, duration, name)")
    a = p.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    c = bench.CONFIGS[a.config]
    dims, ranks = c["dims"], c["ranks"]
    host, buf = bench.make_tensor(c, dims, pinned=True)
    dev = buf.cuda()
    ctx = tk.Context(0)
    dt = tk.DeviceTensor.from_torch(dev, dims)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=50, seed=7))

    def step():
        if c["kind"] == "t":
            return ctx.t_hosvd(dt, tk.Truncation(ranks), eng)
        return ctx.st_hosvd(dt, tk.Truncation(ranks), None, eng)

    for _ in range(a.warm):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
        _, rep = step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
    if not ks:
        print("no device activity recorded")
        return
    t0, t1 = ks[0][0], max(k[1] for k in ks)
    # union of busy intervals
    busy, cur_s, cur_e = 0.0, ks[0][0], ks[0][1]
    gaps = []
    prev_name = ks[0][2]
    for s, e, n in ks[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, prev_name, n, cur_e - t0))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
        if e >= cur_e:
            prev_name = n
    busy += cur_e - cur_s
    span = t1 - t0
    print(f"config {a.config}: span {span / 1e3:.3f} ms, device busy {busy / 1e3:.3f} ms "
          f"({100 * busy / span:.1f} %), {len(ks)} activities, idle {(span - busy) / 1e3:.3f} ms "
          f"in {len(gaps)} gaps; engine seconds {rep.seconds * 1e3:.3f} ms")
    def short(n):
        return n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-60:]

    if a.dump:
        for s_, e_, n in ks:
            print(f"  {(s_ - t0) / 1e3:9.4f} ms  {(e_ - s_):8.1f} us  {short(n)}")
    per = {}
    for s_, e_, n in ks:
        k = short(n)
        per[k] = per.get(k, 0.0) + (e_ - s_)
    for k, v in sorted(per.items(), key=lambda x: -x[1]):
        print(f"  {v / 1e3:9.3f} ms  {k}")
    for g, before, after, at in sorted(gaps, reverse=True)[:a.gaps]:
        print(f"  gap {g:9.1f} us at {at / 1e3:8.3f} ms  after {before[:48]:48s} before {after[:48]}")


if __name__ == "__main__":
    main()
