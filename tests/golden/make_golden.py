"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libfmp_ref.so, i.e. the
reference sources under /root/reference compiled by oracle/Makefile):

    python tests/golden/make_golden.py

Every array comes from the unmodified reference library through
oracle/ref_capi.cpp; nothing here is computed by this repository's code.
The recipes follow the reference's own tests (cited per block).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
if "--text" not in sys.argv:
    from oracle import Oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    import numpy as np
    R = Oracle("reference")
    assert R.impl() == "reference"
    g = {}
    # random.cpp: engine outputs, seeds, gaussians, samples (test_random.cpp:23-74)
    for s in (0, 1, 5, 42, 5489):
        g[f"rng_u64_{s}"] = R.rng_u64(s, 32)
        g[f"rng_cg_{s}"] = R.rng_complex_gaussian(s, 16)
        g[f"rng_sample_{s}"] = R.rng_sample(s, 100, 13)
    g["derive_seed"] = np.array([[b, i, R.derive_seed(b, i)] for b in (0, 1, 7, 60, 2024)
                                 for i in (0, 1, 2, 9, 1 << 40)], dtype=np.uint64)
    # kernels (test_kernel.cpp:41-107) at the reference test sizes and the config sizes
    ker_cases = [(k, n, m, seed) for k in ("fourier", "hadamard")
                 for (n, m, seed) in ((4, 2, 1), (16, 4, 2), (64, 16, 3), (128, 32, 5),
                                      (1024, 256, 11), (4096, 1024, 13))]
    for i, (kind, n, m, seed) in enumerate(ker_cases):
        om = R.make_row_selection(n, m, seed)
        c, vals, vidx = R.compute_kernel(kind, n, om)
        g[f"ker{i}_meta"] = np.array([0 if kind == "fourier" else 1, n, m, seed], np.uint64)
        g[f"ker{i}_omega"] = om
        g[f"ker{i}_c"] = c
        g[f"ker{i}_values"] = vals
        g[f"ker{i}_vidx"] = vidx
    g["ker_count"] = np.array([len(ker_cases)])
    # fast_update vs conventional (test_kernel.cpp:178-219 recipe, own seeds)
    fu = 0
    for kind in ("fourier", "hadamard"):
        for n in (8, 64, 256, 1024):
            for trial in range(3):
                seed = R.derive_seed(60, n * 1000 + trial + (500000 if kind == "hadamard" else 0))
                m = max(2, n // 4)
                k = min(8, m - 1)
                om = R.make_row_selection(n, m, R.derive_seed(seed, 1))
                y = R.rng_complex_gaussian(R.derive_seed(seed, 2), m)
                sup = R.rng_sample(R.derive_seed(seed, 3), n, k)
                co = R.rng_complex_gaussian(R.derive_seed(seed, 4), k)
                h0 = R.apply_adjoint(kind, n, om, y)
                h = R.fast_update(kind, n, om, h0, sup, co, symmetry=False)
                g[f"fu{fu}_meta"] = np.array([0 if kind == "fourier" else 1, n, m], np.uint64)
                g[f"fu{fu}_omega"], g[f"fu{fu}_y"], g[f"fu{fu}_h0"] = om, y, h0
                g[f"fu{fu}_support"], g[f"fu{fu}_coeffs"], g[f"fu{fu}_h"] = sup, co, h
                fu += 1
    g["fu_count"] = np.array([fu])
    # OMP solves: config-1 shape (Hadamard 1024/256/16, real N(0,1)), the two
    # exact-tie seeds (test_solvers.cpp:188-208), the adaptive switch case
    # (test_solvers.cpp:210-234), and one config-2 shaped Fourier signal
    solves = []
    for b in range(4):
        om = R.make_row_selection(1024, 256, R.derive_seed(1, 1 << 40))
        x, y = R.make_real_instance("hadamard", 1024, om, 16, R.derive_seed(1, b))
        solves.append(("hadamard", 1024, om, y, 16, 1e-9 * np.linalg.norm(y)))
    for seed in (4898724841501167528, 14945121902286664584):
        om = R.make_row_selection(256, 16, R.derive_seed(seed, 1))
        x, y, e = R.make_instance("hadamard", 256, om, 8, 0.05, seed)
        solves.append(("hadamard", 256, om, y, 8, 1e-9 * np.linalg.norm(y)))
    om = R.make_row_selection(64, 32, 41)
    x, y, e = R.make_instance("fourier", 64, om, 10, 0.0, 42)
    solves.append(("fourier", 64, om, y, 10, 0.0))
    om = R.make_row_selection(4096, 1024, R.derive_seed(2, 1 << 40))
    x, y, e = R.make_instance("fourier", 4096, om, 64, 0.0, R.derive_seed(2, 0))
    solves.append(("fourier", 4096, om, y, 64, 1e-9 * np.linalg.norm(y)))
    for i, (kind, n, om, y, T, tol) in enumerate(solves):
        g[f"omp{i}_meta"] = np.array([0 if kind == "fourier" else 1, n, len(om), T], np.uint64)
        g[f"omp{i}_tol"] = np.array([tol])
        g[f"omp{i}_omega"], g[f"omp{i}_y"] = om, y
        for mode in ("conventional", "fast", "adaptive"):
            r = R.omp_solve(kind, n, om, y, T, tol, mode=mode, record=False)
            g[f"omp{i}_{mode}_support"] = r.support
            g[f"omp{i}_{mode}_coeffs"] = r.coeffs
            g[f"omp{i}_{mode}_scalars"] = np.array([r.iterations_run, r.residual_norm,
                                                    float(r.rank_deficient_abort)])
            g[f"omp{i}_{mode}_modes"] = np.array(r.mode_used, np.int32)
    g["omp_count"] = np.array([len(solves)])
    # CoSaMP (solvers.cpp:413-544): the noiseless-recovery and edge-case
    # recipes of test_solvers.cpp:236-277 (own seeds for the noisy trials,
    # the acceptance anchor shape of acceptance.cpp:198-205)
    cos = []
    for kind in ("fourier", "hadamard"):
        om = R.make_row_selection(64, 32, 51)
        x, y, e = R.make_instance(kind, 64, om, 4, 0.0, 52)
        cos.append((kind, 64, om, y, 4, 8, 1e-9 * np.linalg.norm(y)))
        for trial in range(3):
            seed = R.derive_seed(80, trial)
            om = R.make_row_selection(128, 64, R.derive_seed(seed, 1))
            x, y, e = R.make_instance(kind, 128, om, 4, 0.05, seed)
            cos.append((kind, 128, om, y, 4, 6, 1e-9 * np.linalg.norm(y)))
    om = R.make_row_selection(64, 8, 61)
    x, y, e = R.make_instance("fourier", 64, om, 4, 0.0, 62)
    cos.append(("fourier", 64, om, y, 4, 6, 0.0))  # rank-deficient abort
    om = R.make_row_selection(8192, 64, 55)
    x, y, e = R.make_instance("fourier", 8192, om, 4, 0.0, 56)
    cos.append(("fourier", 8192, om, y, 4, 6, 0.0))
    for i, (kind, n, om, y, k, T, tol) in enumerate(cos):
        g[f"cos{i}_meta"] = np.array([0 if kind == "fourier" else 1, n, len(om), k, T], np.uint64)
        g[f"cos{i}_tol"] = np.array([tol])
        g[f"cos{i}_omega"], g[f"cos{i}_y"] = om, y
        for mode in ("conventional", "fast"):
            r, sh = R.cosamp_solve(kind, n, om, y, k, T, tol, mode=mode)
            g[f"cos{i}_{mode}_support"] = r.support
            g[f"cos{i}_{mode}_coeffs"] = r.coeffs
            g[f"cos{i}_{mode}_scalars"] = np.array([r.iterations_run, r.residual_norm,
                                                    float(r.rank_deficient_abort)])
            hist = np.zeros((T, k), np.uint64)
            for t, row in enumerate(sh):
                hist[t, : len(row)] = row
            g[f"cos{i}_{mode}_history"] = hist
    g["cos_count"] = np.array([len(cos)])
    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_golden.npz"))
    # the reference library links libstdc++ statically (the image's $CXX);
    # its iostreams must not meet the libstdc++ numpy loads: separate process
    subprocess.run([sys.executable, os.path.abspath(__file__), "--text"], check=True)


def text_fixtures():
    """Instance / result / cost-CSV text written by the reference's
    save_instance, save_result and CostReport::write_csv."""
    import ctypes as C
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libfmp_ref.so"))
    L.fmpo_ref_instance_text.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                         C.c_uint64, C.c_char_p, C.c_uint64,
                                         C.POINTER(C.c_uint64)]
    L.fmpo_ref_result_text.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_uint64,
                                       C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
    L.fmpo_ref_counts_text.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    cases = [("fourier", 64, 32, 4, 0.0, 11), ("hadamard", 64, 32, 4, 0.05, 12),
             ("fourier", 256, 64, 8, 0.05, 13), ("hadamard", 1024, 256, 16, 0.0, 14)]
    for kind, n, m, k, noise, seed in cases:
        buf = C.create_string_buffer(1 << 22)
        ln = C.c_uint64()
        assert L.fmpo_ref_instance_text(0 if kind == "fourier" else 1, n, m, k, noise, seed, buf,
                                        len(buf), C.byref(ln)) == 0
        inst = buf.value
        stem = f"{kind}_{n}_{m}_{k}_{seed}"
        with open(os.path.join(OUT, f"instance_{stem}.txt"), "wb") as f:
            f.write(inst)
        cbuf = C.create_string_buffer(1 << 20)
        assert L.fmpo_ref_counts_text(inst, cbuf, len(cbuf), C.byref(ln)) == 0
        with open(os.path.join(OUT, f"counts_{stem}.txt"), "wb") as f:
            f.write(cbuf.value)
        for mode, code in (("conventional", 0), ("fast", 1)):
            rb = C.create_string_buffer(1 << 20)
            cb = C.create_string_buffer(1 << 20)
            assert L.fmpo_ref_result_text(inst, code, rb, len(rb), C.byref(ln), cb, len(cb),
                                          C.byref(ln)) == 0
            with open(os.path.join(OUT, f"result_{stem}_{mode}.txt"), "wb") as f:
                f.write(rb.value)
            with open(os.path.join(OUT, f"costs_{stem}_{mode}.csv"), "wb") as f:
                f.write(cb.value)
    print("wrote text fixtures")


if __name__ == "__main__":
    if "--text" in sys.argv:
        text_fixtures()
    else:
        main()
