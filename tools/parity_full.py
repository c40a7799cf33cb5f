#!/usr/bin/env python3
"""Full-size parity of the five BASELINE configs (SURVEY §8(c) last bullet,
§8(d)): the B200 path against the compiled, unmodified
reference (oracle/_ref, `tenkit::t_hosvd` / `st_hosvd`, hosvd.cpp:74-191) on
IDENTICAL bytes.

Per config, in one process:
  1. synthesise the config tensor once (csrc/synth.cpp, seeded);
  2. decompose it on the GPU through the public API (host tensor in);
  3. check the st core shortcut (hosvd.cpp:176-178) against an explicit TTM
     chain A x_n U_n^T of the same tensor on the GPU;
  4. write it as TNSR, free it, and let the reference read it back with its own
     read_tnsr and decompose it with all host threads (the file is the only
     channel between the two arms);
  5. record iterations per mode, |d rel err|, principal-angle sines, core
     mode-n spectra, orthonormality, every stop decision's margin
     |res_{k-1} - res_k| / ||A_work|| against eta, and the CPU times.

  python tools/parity_full.py --config 3 [--scale 1.0] [--out file.json]

--scale s < 1 shrinks every extent by s (ranks kept), for a quicker run.
Test/measurement infrastructure: imports tests/oracles (the checker).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402  (CONFIGS, ALS_SEED, MAX_ITERS)


def write_tnsr(path, a):
    """TNSR v1 (io.cpp:19-24,131-139): magic, u32 version, u32 order,
    u64 extents, f64 payload in column-major order."""
    with open(path, "wb") as f:
        f.write(b"TNSR")
        f.write(np.array([1, a.ndim], dtype="<u4").tobytes())
        f.write(np.array(a.shape, dtype="<u8").tobytes())
        flat = a.reshape(-1, order="F")
        step = 1 << 26
        for s in range(0, flat.size, step):
            f.write(flat[s:s + step].astype("<f8", copy=False).tobytes())


def decisions(history, norm, eta):
    """The stop rule's quantities d_k = |res_{k-1} - res_k| / ||A|| (als.cpp:
    124-150), res_0 = ||A||, and their ratios to eta (continue while > 1)."""
    prev, out = norm, []
    for h in history:
        d = abs(prev - h) / norm
        out.append(d / eta)
        prev = h
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(cfg_id, scale, tmpdir, threads):
    import paper_2004_02583_b200 as tk
    from oracles import Ref
    from parity import (ANGLE_TOL, CORE_SV_REL_TOL, REL_ERR_ABS_TOL, core_mode_spectra,
                        ortho_defect, principal_sine)

    c = bench.CONFIGS[cfg_id]
    dims = [max(int(round(d * scale)), r + 1) for d, r in zip(c["dims"], c["ranks"])]
    ranks = c["ranks"]
    st = c["kind"] == "st"
    rec = {"config": cfg_id, "kind": c["kind"], "dims": dims, "ranks": ranks, "eta": c["eta"],
           "max_iters": bench.MAX_ITERS, "als_seed": bench.ALS_SEED, "synth_seed": c["seed"],
           "alpha": c["alpha"], "nu": c["nu"], "scale": scale}
    t0 = time.time()
    a = tk.synth_tucker(dims, ranks, c["alpha"], c["nu"], c["seed"]).reshape(dims, order="F")
    rec["synth_s"] = time.time() - t0
    norm_a = float(np.sqrt(np.dot(a.reshape(-1, order="F"), a.reshape(-1, order="F"))))

    # ---- GPU ---------------------------------------------------------------
    ctx = tk.Context(0)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=bench.MAX_ITERS,
                                                seed=bench.ALS_SEED))
    t0 = time.time()
    if st:
        g_tk, g_rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
    else:
        g_tk, g_rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    rec["gpu_call_s"] = time.time() - t0
    rec["gpu_report_seconds"] = g_rep.seconds
    # the core against an explicit TTM chain of the same tensor (st: the
    # R^ R^T shortcut of hosvd.cpp:176-178; t: the first-step identity, §5)
    explicit = ctx.multi_mode_product(a, [(u.T, n + 1) for n, u in enumerate(g_tk.factors)])
    rec["core_vs_explicit_ttm_rel"] = float(np.max(np.abs(explicit - g_tk.core)) /
                                            np.max(np.abs(explicit)))
    del explicit
    # ||working tensor|| at each st position: A x_m U_m^T over the modes
    # processed before it (the stop rule's denominator, als.cpp:102)
    work_norms = [norm_a]
    if st:
        done = []
        for m in [pm.mode for pm in g_rep.per_mode][:-1]:
            done.append((g_tk.factors[m - 1].T, m))
            w = ctx.multi_mode_product(a, sorted(done, key=lambda x: x[1]))
            work_norms.append(float(np.linalg.norm(w)))
            del w
    ctx.close()
    del ctx

    # ---- reference (reads the same bytes back from a TNSR file) -------------
    path = os.path.join(tmpdir, f"parity_c{cfg_id}.tnsr")
    t0 = time.time()
    write_tnsr(path, a)
    rec["tnsr_write_s"] = time.time() - t0
    del a
    ref = Ref()
    ref.set_threads(threads)
    try:
        r_res, r_call_s = ref.hosvd_als_tnsr(path, dims, ranks, sequential=st, eta=c["eta"],
                                            max_iters=bench.MAX_ITERS, seed=bench.ALS_SEED)
    finally:
        os.unlink(path)
    rec["cpu"] = {"call_s": r_call_s, "report_seconds": r_res.seconds, "threads": threads,
                  "cpu_model": cpu_model(), "nproc": os.cpu_count()}

    # ---- compare ---------------------------------------------------------------
    modes = []
    for pos, (gm, rm) in enumerate(zip(g_rep.per_mode, r_res.per_mode)):
        g_hist, r_hist = gm.als.residual_history, rm.residual_history
        nrm = work_norms[pos] if st else norm_a
        r_ratio = decisions(r_hist, nrm, c["eta"])
        g_ratio = decisions(g_hist, nrm, c["eta"])
        closest = min(r_ratio, key=lambda x: abs(np.log(max(x, 1e-300))))
        modes.append({
            "mode": rm.mode, "gpu_mode": gm.mode,
            "iters_ref": rm.iterations, "iters_gpu": gm.als.iterations,
            "status_ref": "converged" if rm.status == 0 else "max_iters_reached",
            "status_gpu": gm.als.status,
            "history_ref": r_hist, "history_gpu": g_hist,
            "history_max_rel_diff": float(max((abs(x - y) / max(abs(y), 1e-300)
                                              for x, y in zip(g_hist, r_hist)), default=0.0)),
            "work_norm": nrm,
            "decision_ratio_ref": r_ratio, "decision_ratio_gpu": g_ratio,
            "closest_decision_ratio": closest,
            "seconds_ref": rm.seconds, "seconds_gpu": gm.seconds,
        })
    angles = [principal_sine(g, r) for g, r in zip(g_tk.factors, r_res.factors)]
    spectra_g = core_mode_spectra(np.asarray(g_tk.core))
    spectra_r = core_mode_spectra(np.asarray(r_res.core))
    sv_rel = [float(np.max(np.abs(sg - sr)) / np.max(np.abs(sr))) for sg, sr in zip(spectra_g, spectra_r)]
    rec.update({
        "modes": modes,
        "iters_equal": all(m["iters_ref"] == m["iters_gpu"] and m["mode"] == m["gpu_mode"] for m in modes),
        "rel_err_gpu": g_rep.relative_residual, "rel_err_ref": r_res.relative_residual,
        "rel_err_abs_diff": abs(g_rep.relative_residual - r_res.relative_residual),
        "principal_sines": angles, "max_principal_sine": max(angles),
        "core_sv_rel_diff_per_mode": sv_rel, "core_sv_rel_diff": max(sv_rel),
        "ortho_defect_gpu": [ortho_defect(u) for u in g_tk.factors],
        "ortho_defect_ref": [ortho_defect(u) for u in r_res.factors],
        "tolerances": {"rel_err_abs": REL_ERR_ABS_TOL, "principal_sine": ANGLE_TOL,
                       "core_sv_rel": CORE_SV_REL_TOL},
    })
    rec["pass"] = bool(rec["iters_equal"] and rec["rel_err_abs_diff"] <= REL_ERR_ABS_TOL and
                       rec["max_principal_sine"] <= ANGLE_TOL and
                       rec["core_sv_rel_diff"] <= CORE_SV_REL_TOL)
    return rec


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, required=True)
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--tmpdir", default="/tmp")
    p.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    p.add_argument("--out", default=None)
    args = p.parse_args()
    rec = run(args.config, args.scale, args.tmpdir, args.threads)
    s = json.dumps(rec)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")
    short = {k: rec[k] for k in ("config", "dims", "pass", "iters_equal", "rel_err_abs_diff",
                                 "max_principal_sine", "core_sv_rel_diff", "core_vs_explicit_ttm_rel")}
    short["closest_decision_ratio"] = [m["closest_decision_ratio"] for m in rec["modes"]]
    short["iters"] = [(m["mode"], m["iters_ref"], m["iters_gpu"]) for m in rec["modes"]]
    short["cpu_s"] = rec["cpu"]["call_s"]
    print(json.dumps(short))
    return 0 if rec["pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
