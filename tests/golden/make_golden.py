"""Generate tests/golden/*.npz from the reference itself (oracle/_ref/libcoru_ref.so, compiled from
/root/reference/proj/include by oracle/Makefile). Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The cases are the reference's own hot-path tests (proj/tests/test_corutv.cpp, test_matcore.cpp),
with their matrices built by the reference's generators (testgen.hpp) and seeds. The fixtures pin
(1) the plain-C oracle restatement bit-for-bit and (2) the GPU path within tolerance, on machines
where the reference tree is absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402

R = Reference()


def exact_rank_matrix(m, n, r, seed, stream=0):
    # test_corutv.cpp:16-19: matmul(gaussian(m, r, substream(seed, 0)), gaussian(n, r, substream(seed, 1))^T)
    g1 = R.gaussian(m, r, seed, stream + 0)
    g2 = R.gaussian(n, r, seed, stream + 1)
    return R.matmul(g1, np.ascontiguousarray(g2.T))


def main():
    cases = []  # (name, A, ell, q, seed, stream)
    cases.append(("exact_rank_30x20_r5", exact_rank_matrix(30, 20, 5, 3), 5, 0, 4, 0))      # :38-42
    fd80 = R.gen_fast_decay(80, 8, 5)
    cases.append(("fast_decay_80_q0", fd80, 20, 0, 6, 0))                                   # :44-55
    cases.append(("fast_decay_80_q2", fd80, 20, 2, 6, 0))
    cases.append(("fast_decay_60_q1", R.gen_fast_decay(60, 6, 7), 15, 1, 8, 0))             # :57-65
    nl400 = R.gen_noisy_lowrank(400, 20, 0.01, 12345)
    cases.append(("noisy_lowrank_400_q0_s1000", nl400, 40, 0, 1000, 0))                     # :67-75
    cases.append(("noisy_lowrank_400_q2", nl400, 40, 2, 2024, 0))                            # :77-85
    cases.append(("wide_20x35_ulv", exact_rank_matrix(20, 35, 4, 11), 8, 1, 12, 0))         # :98-108
    cases.append(("fast_decay_50_q1", R.gen_fast_decay(50, 5, 13), 12, 1, 14, 0))           # :110-116
    d = np.zeros((6, 5)); d[0, 0], d[1, 1], d[2, 2] = 5.0, 3.0, 1.0
    cases.append(("diag531_6x5", d, 3, 2, 15, 0))                                            # :133-144
    cases.append(("rank1_12x9", exact_rank_matrix(12, 9, 1, 16), 2, 0, 17, 0))              # :146-148
    fd120 = R.gen_fast_decay(120, 5, 26)
    cases.append(("fast_decay_120_q0", fd120, 30, 0, 27, 0))                                 # :198-206
    cases.append(("fast_decay_120_q6", fd120, 30, 6, 27, 0))
    nl150 = R.gen_noisy_lowrank(150, 10, 0.01, 23)
    cases.append(("noisy_lowrank_150_q0", nl150, 20, 0, 200, 0))                             # :208-220
    cases.append(("noisy_lowrank_150_q2", nl150, 20, 2, 200, 0))

    out = {}
    names = []
    mats = {}  # each distinct input stored once
    for name, a, ell, q, seed, stream in cases:
        f = R.corutv(a, ell, q, 0, seed, stream)
        names.append(name)
        key = next((k for k, v in mats.items() if v.shape == a.shape and np.array_equal(v, a)), None)
        if key is None:
            key = f"mat{len(mats)}"
            mats[key] = a
            out[f"A/{key}"] = a
        out[f"{name}/Akey"] = np.array(key)
        out[f"{name}/params"] = np.array([ell, q, seed, stream], np.int64)
        out[f"{name}/U"], out[f"{name}/T"], out[f"{name}/V"] = f.u, f.t, f.v
        out[f"{name}/flags"] = np.array([f.lower, f.conditioning_warning], np.int64)
    # sketch_bases (test_corutv.cpp:61) on fast_decay_60
    q1, q2, c1, c2p, w = R.sketch_bases(R.gen_fast_decay(60, 6, 7), 15, 1, 8, 0)
    out["sketch_60/Q1"], out["sketch_60/Q2"], out["sketch_60/C1"], out["sketch_60/C2prev"] = q1, q2, c1, c2p
    out["sketch_60/flag"] = np.array([w], np.int64)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "corutv_ref_cases.npz"), **out)

    # RNG / QR / QRCP known answers (test_matcore.cpp:21-117, 207-230)
    kat = {}
    kat["xoshiro_42_0"] = R.xoshiro_words(42, 0, 64)
    kat["xoshiro_0_0"] = R.xoshiro_words(0, 0, 16)  # all-zero SplitMix guard path (rng.hpp:47-48)
    kat["gaussian_4x4_1_0"] = R.gaussian(4, 4, 1, 0)
    kat["gaussian_4x4_1_1"] = R.gaussian(4, 4, 1, 1)
    kat["gaussian_7x9_42_3"] = R.gaussian(7, 9, 42, 3)
    kat["gaussian_100x100_42_0"] = R.gaussian(100, 100, 42, 0)
    kat["gaussian_1x5_7_0"] = R.gaussian(1, 5, 7, 0)  # odd count: the spare is dropped
    g = R.gaussian(50, 20, 31, 0)
    kat["qr_in"] = g
    kat["qr_q"], kat["qr_r"] = R.householder_qr(g)
    q, r = R.householder_qr(np.array([[3.0], [4.0]]))
    kat["qr34_q"], kat["qr34_r"] = q, r
    rd = np.zeros((5, 3))
    for i in range(5):
        rd[i, 0] = rd[i, 2] = i + 1.0
    kat["qr_rankdef_in"] = rd
    kat["qr_rankdef_q"], kat["qr_rankdef_r"] = R.householder_qr(rd)
    dd = np.diag([1.0, 5.0, 3.0])
    kat["qrcp_diag_q"], kat["qrcp_diag_r"], kat["qrcp_diag_perm"] = R.qrcp(dd)
    u9, v6 = R.gaussian(9, 1, 41, 0), R.gaussian(6, 1, 41, 1)
    r1 = R.matmul(u9, np.ascontiguousarray(v6.T))
    kat["qrcp_rank1_in"] = r1
    kat["qrcp_rank1_q"], kat["qrcp_rank1_r"], kat["qrcp_rank1_perm"] = R.qrcp(r1)
    for trial in range(12):                                        # test_matcore.cpp:102-117
        m = 8 + (trial * 7) % 30
        n = 2 + (trial * 5) % (min(m, 15) - 1)
        a = R.gaussian(m, n, trial, 7)
        kat[f"qrcp_trial{trial}_in"] = a
        kat[f"qrcp_trial{trial}_q"], kat[f"qrcp_trial{trial}_r"], kat[f"qrcp_trial{trial}_perm"] = R.qrcp(a)
    np.savez_compressed(os.path.join(HERE, "kernels_ref_kat.npz"), **kat)
    print("wrote", len(names), "corutv cases and", len(kat), "kernel KAT arrays")
    approx_fixtures(cases)
    baseline_fixtures()


def baseline_fixtures():
    """SOR-SVD / TSR-SVD (baselines.hpp:43-71) on the inputs of proj/tests/test_baselines.cpp."""
    bl = {}
    tsr = [("tsr_rank1_50x30", R.matmul(R.gaussian(50, 1, 17, 0), np.ascontiguousarray(R.gaussian(30, 1, 17, 1).T)),
            2, 18, 0),                                                                          # :57-66
           ("tsr_fast_decay_70", R.gen_fast_decay(70, 7, 19), 14, 20, 3),                      # :68-79
           ("tsr_noisy_200", R.gen_noisy_lowrank(200, 10, 0.1, 21), 20, 400, 0),               # :81-97
           ("tsr_wide_40x90", R.gaussian(40, 90, 31, 2) * (0.9 ** np.arange(90)), 12, 32, 0)]
    for name, a, ell, seed, stream in tsr:
        u, s, v, conv = R.tsr_svd(a, ell, seed, stream)
        bl[f"{name}/A"], bl[f"{name}/params"] = a, np.array([ell, seed, stream], np.int64)
        bl[f"{name}/U"], bl[f"{name}/S"], bl[f"{name}/V"] = u, s, v
        bl[f"{name}/conv"] = np.array([conv], np.int64)
    er = R.matmul(R.gaussian(25, 5, 22, 0), np.ascontiguousarray(R.gaussian(18, 5, 22, 1).T))
    sor = [("sor_exact_rank_25x18", er, 5, 8, 0, 23, 0),                                      # :99-104
           ("sor_fast_decay_60_k12", R.gen_fast_decay(60, 6, 24), 12, 12, 0, 25, 0),            # :106-112
           ("sor_noisy_200", R.gen_noisy_lowrank(200, 10, 0.01, 26), 10, 20, 0, 500, 0),        # :114-124
           ("sor_noisy_100", R.gen_noisy_lowrank(100, 10, 0.1, 5), 10, 20, 0, 6, 0),            # :45-55
           ("sor_q2_90x60", R.gen_fast_decay(90, 9, 41)[:, :60].copy(), 6, 15, 2, 42, 1),
           ("sor_wide_30x50", R.gaussian(30, 50, 43, 0) * (0.85 ** np.arange(50)), 4, 9, 1, 44, 0)]
    for name, a, k, ell, q, seed, stream in sor:
        bl[f"{name}/A"], bl[f"{name}/params"] = a, np.array([k, ell, q, seed, stream], np.int64)
        bl[f"{name}/L"] = R.sor_svd(a, k, ell, q, seed, stream)
    bl["tsr_names"] = np.array([t[0] for t in tsr])
    bl["sor_names"] = np.array([t[0] for t in sor])
    np.savez_compressed(os.path.join(HERE, "baselines_ref_cases.npz"), **bl)
    print("wrote", len(tsr), "tsr_svd and", len(sor), "sor_svd cases")


def approx_fixtures(cases):
    """DVariant::approx (corutv.hpp:91-92) and its pinv core (svd.hpp:31-187)."""
    ap = {}
    anames = []
    er = exact_rank_matrix(40, 30, 6, 9)                                                      # test_corutv.cpp:87-96
    acases = [("approx_exact_rank_40x30_q0", er, 10, 0, 10, 0), ("approx_exact_rank_40x30_q2", er, 10, 2, 10, 0)]
    pick = {"fast_decay_80_q0", "fast_decay_80_q2", "wide_20x35_ulv", "noisy_lowrank_150_q0",
            "noisy_lowrank_150_q2", "fast_decay_120_q0", "diag531_6x5", "rank1_12x9"}
    acases += [("approx_" + c[0],) + c[1:] for c in cases if c[0] in pick]
    for name, a, ell, q, seed, stream in acases:
        f = R.corutv(a, ell, q, 1, seed, stream)
        anames.append(name)
        ap[f"{name}/A"] = a
        ap[f"{name}/params"] = np.array([ell, q, seed, stream], np.int64)
        ap[f"{name}/U"], ap[f"{name}/T"], ap[f"{name}/V"] = f.u, f.t, f.v
        ap[f"{name}/flags"] = np.array([f.lower, f.conditioning_warning], np.int64)
    ap["names"] = np.array(anames)
    # pinv / square Jacobi SVD known answers (test_matcore.cpp:119-205) and the cores the approx
    # variant actually inverts: Q2^T·C2prev from the reference's own sketch_bases.
    sq = {}
    sq["diag3m2"] = np.array([[3.0, 0.0], [0.0, -2.0]])
    sq["swap2"] = np.array([[0.0, 1.0], [1.0, 0.0]])
    d2 = np.zeros((2, 2)); d2[0, 0] = 2.0
    sq["diag2_0"] = d2
    sq["zero3"] = np.zeros((3, 3))
    stream = 0
    for m in range(1, 5):                                                                    # :138-150 (square)
        sq[f"gauss{m}x{m}"] = R.gaussian(m, m, 77, stream + 5 * (m - 1))
    for trial, n in enumerate((7, 12, 25, 40)):
        sq[f"gauss{n}_t{trial}"] = R.gaussian(n, n, trial + 1, 3)
    u, v = R.gaussian(6, 2, 9, 0), R.gaussian(6, 2, 9, 1)                                    # :170-176
    sq["rank2_6"] = R.matmul(u, np.ascontiguousarray(v.T))
    g = R.gaussian(30, 30, 5, 5)
    sq["graded30"] = g * (10.0 ** -(np.arange(30) / 2.0))
    for name, a, ell, q, seed, stream in acases[:2] + [c for c in acases if c[0] in ("approx_fast_decay_80_q2", "approx_noisy_lowrank_150_q0")]:
        if a.shape[0] < a.shape[1]:
            continue
        q1, q2, c1, c2p, _ = R.sketch_bases(a, ell, q, seed, stream)
        sq[f"core_{name}"] = R.matmul(np.ascontiguousarray(q2.T), c2p)
    for k, a in sq.items():
        ap[f"pinv/{k}/in"] = a
        ap[f"pinv/{k}/out"] = R.pinv(a)
        uu, ss, vv, conv = R.svd(a)
        ap[f"pinv/{k}/u"], ap[f"pinv/{k}/s"], ap[f"pinv/{k}/v"] = uu, ss, vv
        ap[f"pinv/{k}/conv"] = np.array([conv], np.int64)
    ap["pinv_names"] = np.array(list(sq))
    np.savez_compressed(os.path.join(HERE, "approx_ref_cases.npz"), **ap)
    print("wrote", len(anames), "approx corutv cases and", len(sq), "pinv cases")


def rpca_instance_rect(m, n, r, nnz, amp, seed):
    """Rectangular restatement of gen_rpca_instance (testgen.hpp:86-109) for the non-square cases:
    L = G1·G2^T from the reference's gaussian sub-streams, nnz entries ±amp at seeded positions."""
    g1 = R.gaussian(m, r, seed, 0)
    g2 = R.gaussian(n, r, seed, 1)
    low = R.matmul(g1, np.ascontiguousarray(g2.T))
    rng = np.random.default_rng(seed)
    sp = np.zeros(m * n)
    idx = rng.choice(m * n, nnz, replace=False)
    sp[idx] = np.where(rng.random(nnz) < 0.5, amp, -amp)
    return low + sp.reshape(m, n)


def rpca_fixtures(full=True):
    """alm_rpca with the CoR-UTV inner (rpca.hpp:95-169): the reference's instances (test_cli.cpp:168-183
    gen --family rpca --n 60 --k 4 --s 180 --amp 80 --seed 21; acceptance.cpp:204-220,394 criterion 7)."""
    out = {}
    names = []
    m60 = R.gen_rpca_instance(60, 4, 180, 80.0, 21)[0]
    tall = rpca_instance_rect(90, 50, 3, 150, 60.0, 5)
    wide = np.ascontiguousarray(rpca_instance_rect(90, 50, 3, 150, 60.0, 6).T)
    cases = [
        ("n60_soft_ell8", m60, dict(corutv_ell=8, corutv_q=1, thresholding=0)),
        ("n60_hard_ell8", m60, dict(corutv_ell=8, corutv_q=1, thresholding=1)),
        ("n60_soft_predict", m60, dict(corutv_ell=0, corutv_q=1, thresholding=0)),
        ("n60_hard_q0_maxit3", m60, dict(corutv_ell=8, corutv_q=0, thresholding=1, max_iter=3)),
        ("tall90x50_soft_ell6", tall, dict(corutv_ell=6, corutv_q=1, thresholding=0)),
        ("tall90x50_hard_ell6", tall, dict(corutv_ell=6, corutv_q=2, thresholding=1)),
        ("wide50x90_hard_ell6", wide, dict(corutv_ell=6, corutv_q=1, thresholding=1)),
        ("wide50x90_soft_ell6_mu0", wide, dict(corutv_ell=6, corutv_q=1, thresholding=0, mu0=0.01)),
    ]
    if full:
        m400 = R.gen_rpca_instance(400, 20, 8000, 80.0, 2024)
        cases.append(("acc7_n400_r20_soft_ell40", m400[0], dict(corutv_ell=40, corutv_q=1, thresholding=0)))
        out["acc7_n400_r20_soft_ell40/S_true"] = m400[2]
    for name, mat, kw in cases:
        r = R.alm_rpca(mat, seed=2, stream=0, **kw)
        names.append(name)
        out[f"{name}/M"] = mat
        out[f"{name}/L"] = r["l"]
        out[f"{name}/S"] = r["s"]
        out[f"{name}/residuals"] = r["residuals"]
        cfg = dict(lambda_=0.0, mu0=0.0, rho=1.5, mu_bar=0.0, tol=1e-5, max_iter=50, corutv_ell=0, corutv_q=1,
                   thresholding=0)
        cfg.update(kw)
        out[f"{name}/cfg"] = np.array([cfg["lambda_"], cfg["mu0"], cfg["rho"], cfg["mu_bar"], cfg["tol"],
                                       cfg["max_iter"], cfg["corutv_ell"], cfg["corutv_q"], cfg["thresholding"]])
        out[f"{name}/out"] = np.array([r["iterations"], r["rank_l"], r["s_l0"], r["converged"], r["ell_clamped"]],
                                      np.int64)
        print(name, "it", r["iterations"], "rank", r["rank_l"], "s_l0", r["s_l0"], "conv", r["converged"])
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "rpca_ref_cases.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "rpca":
        rpca_fixtures()
        sys.exit(0)
    main()


def bin_fixtures():
    """CORU binary files written by the reference's write_matrix_bin (io.hpp:67-77)."""
    R.write_matrix_bin(os.path.join(HERE, "ref_matrix_3x2.bin"),
                       np.array([[1.5, -2.0], [3.25, np.pi], [1e-300, -0.0]]))
    R.write_matrix_bin(os.path.join(HERE, "ref_gaussian_64x24.bin"), R.gaussian(64, 24, 5, 0))
