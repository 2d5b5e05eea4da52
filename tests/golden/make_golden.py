"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and oracle/_ref/
libptycho_ref.so is built):   python tests/golden/make_golden.py

Every fixture is produced by the reference's own code (through the C veneer
oracle/ref_capi.cpp) on small seeded ref-mode problems (binary windows,
full-field n x n FFTs), so the committed vectors pin the oracle and the GPU
path on the GPU box, where /root/reference does not exist.  Inputs are seeded
numpy draws; outputs are the reference's results, stored at full float64
precision.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ptgo  # noqa: E402


def rf(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return scale * (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))


def main():
    assert ptgo.has_reference(), "build oracle/_ref/libptycho_ref.so first (make -C oracle)"
    out = {}

    # kernels.cpp:34-85 -- fft2 known answers
    for n in (1, 2, 8, 32):
        x = rf(n, 100 + n)
        out[f"fft_in_{n}"] = x
        out[f"fft_fwd_{n}"] = ptgo.ref_fft2(x, False)
        out[f"fft_inv_{n}"] = ptgo.ref_fft2(x, True)

    # objectives.cpp:106-118 on two ref-mode geometries, both metrics, with shift
    for tag, (n, w, s) in {"a": (16, 8, 4), "b": (32, 16, 8)}.items():
        win = ptgo.ref_raster(n, w, s)
        pos = win[:, :2].copy()
        zt, z, v = rf(n, 11), rf(n, 12), rf(n, 13, 0.1)
        data = ptgo.ref_simulate(n, w, pos, zt)
        out[f"eval_{tag}_geom"] = np.array([n, w, s])
        out[f"eval_{tag}_pos"] = pos
        out[f"eval_{tag}_truth"] = zt
        out[f"eval_{tag}_z"] = z
        out[f"eval_{tag}_v"] = v
        out[f"eval_{tag}_data"] = data
        for m in (0, 1):
            val, g = ptgo.ref_evaluate(m, n, w, pos, data, z, v)
            out[f"eval_{tag}_m{m}_value"] = np.array(val)
            out[f"eval_{tag}_m{m}_grad"] = g
        # projectModulus (objectives.cpp:42-50) for a few windows
        for k in (0, len(pos) // 2, len(pos) - 1):
            out[f"proj_{tag}_{k}"] = ptgo.ref_project_modulus(n, win[k], data[k], z)

    # multigrid.cpp:34-77 transfer operators
    f = rf(16, 21)
    out["xfer_fine"] = f
    out["xfer_restrict"] = ptgo.ref_restrict_field(f)
    out["xfer_prolong"] = ptgo.ref_prolong_field(out["xfer_restrict"])
    d = np.abs(np.random.default_rng(22).normal(size=(3, 16, 16)))
    out["xfer_data"] = d
    out["xfer_restrict_data"] = ptgo.ref_restrict_data(d)

    # solvers: PIE (solvers.cpp:229-265), LBFGS (:87-141), MG/OPT driver (multigrid.cpp:171-227)
    n, w, s = 32, 16, 8
    pos = ptgo.ref_raster(n, w, s)[:, :2].copy()
    data = out["eval_b_data"]
    z0 = rf(n, 31, 0.5)
    r = ptgo.ref_pie(n, w, pos, data, z0, 0.1, 3)
    out["pie_z0"], out["pie_z"], out["pie_hist"] = z0, r.z, r.history
    out["pie_meta"] = np.array([r.value, r.weighted, r.reason])
    r = ptgo.ref_lbfgs(0, n, w, pos, data, z0, v=out["eval_b_v"], max_iters=6)
    out["lbfgs_z"], out["lbfgs_hist"] = r.z, r.history
    out["lbfgs_meta"] = np.array([r.value, r.weighted, r.reason])
    # truncatedNewton (solvers.cpp:143-227): Newton-CG with finite-difference
    # Hessian-vector products, shifted objective, few outer / inner iterations
    r = ptgo.ref_truncated_newton(0, n, w, pos, data, z0, v=out["eval_b_v"], max_iters=4, cg_max_iters=5)
    out["tn_z"], out["tn_hist"] = r.z, r.history
    out["tn_meta"] = np.array([r.value, r.weighted, r.reason])
    # diagnostics (metrics.cpp:67-136) on a reconstruction vs the truth and on a
    # random 40x40 pair (phase maps with a full [-pi, pi] range)
    out["met_a"] = np.array(ptgo.ref_metrics(out["tn_z"], out["eval_b_truth"]))
    out["met_phase_a"] = ptgo.ref_canonical_phase(out["tn_z"])
    rng = np.random.default_rng(77)
    za = rng.normal(size=(40, 40)) + 1j * rng.normal(size=(40, 40))
    zb = za + 0.3 * (rng.normal(size=(40, 40)) + 1j * rng.normal(size=(40, 40)))
    out["met_za"], out["met_zb"] = za, zb
    out["met_b"] = np.array(ptgo.ref_metrics(za, zb))
    out["met_phase_b"] = ptgo.ref_canonical_phase(za)
    # MG/OPT from a non-degenerate start: at z = 1 a binary window's spectrum has
    # exact zeros where the theta(0) = 0 rule makes the gradient depend on FFT
    # rounding, so any other FFT cannot reproduce it
    for depth in (2, 3):
        zs = 1.0 + rf(n, 41, 0.25)
        out[f"mg{depth}_z0"] = zs
        # coarsest solve capped at 10 iterations: 100 LBFGS iterations run into the
        # rounding floor where accept/reject decisions flip between FFT orderings
        r = ptgo.ref_mgopt(0, n, w, s, data, zs, depth, coarsest_max_iters=10, budget=1e9, max_cycles=3)
        out[f"mg{depth}_z"], out[f"mg{depth}_hist"] = r.z, r.history
        out[f"mg{depth}_meta"] = np.array([r.value, r.weighted, r.reason] + r.per_level)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
