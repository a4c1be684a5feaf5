"""Golden fixtures generated from the compiled reference (see make_golden.py)."""
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def corutv_cases():
    z = np.load(os.path.join(HERE, "corutv_ref_cases.npz"))
    out = []
    for name in z["names"]:
        name = str(name)
        ell, q, seed, stream = (int(x) for x in z[f"{name}/params"])
        lower, warn = (bool(x) for x in z[f"{name}/flags"])
        a = z[f"A/{str(z[f'{name}/Akey'])}"]
        out.append(dict(name=name, A=a, ell=ell, q=q, seed=seed, stream=stream, U=z[f"{name}/U"],
                        T=z[f"{name}/T"], V=z[f"{name}/V"], lower=lower, warning=warn))
    return out


def sketch_case():
    z = np.load(os.path.join(HERE, "corutv_ref_cases.npz"))
    a = next(c["A"] for c in corutv_cases() if c["name"] == "fast_decay_60_q1")
    return dict(A=a, ell=15, q=1, seed=8, stream=0, Q1=z["sketch_60/Q1"], Q2=z["sketch_60/Q2"],
                C1=z["sketch_60/C1"], C2prev=z["sketch_60/C2prev"], warning=bool(z["sketch_60/flag"][0]))


def kat():
    return dict(np.load(os.path.join(HERE, "kernels_ref_kat.npz")))


def approx_cases():
    z = np.load(os.path.join(HERE, "approx_ref_cases.npz"))
    out = []
    for name in z["names"]:
        name = str(name)
        ell, q, seed, stream = (int(x) for x in z[f"{name}/params"])
        lower, warn = (bool(x) for x in z[f"{name}/flags"])
        out.append(dict(name=name, A=z[f"{name}/A"], ell=ell, q=q, seed=seed, stream=stream, U=z[f"{name}/U"],
                        T=z[f"{name}/T"], V=z[f"{name}/V"], lower=lower, warning=warn))
    return out


def pinv_cases():
    z = np.load(os.path.join(HERE, "approx_ref_cases.npz"))
    return [dict(name=str(k), A=z[f"pinv/{k}/in"], P=z[f"pinv/{k}/out"], U=z[f"pinv/{k}/u"], S=z[f"pinv/{k}/s"],
                 V=z[f"pinv/{k}/v"], converged=bool(z[f"pinv/{k}/conv"][0])) for k in z["pinv_names"]]


def tsr_cases():
    z = np.load(os.path.join(HERE, "baselines_ref_cases.npz"))
    out = []
    for name in z["tsr_names"]:
        name = str(name)
        ell, seed, stream = (int(x) for x in z[f"{name}/params"])
        out.append(dict(name=name, A=z[f"{name}/A"], ell=ell, seed=seed, stream=stream, U=z[f"{name}/U"],
                        S=z[f"{name}/S"], V=z[f"{name}/V"], converged=bool(z[f"{name}/conv"][0])))
    return out


def sor_cases():
    z = np.load(os.path.join(HERE, "baselines_ref_cases.npz"))
    out = []
    for name in z["sor_names"]:
        name = str(name)
        k, ell, q, seed, stream = (int(x) for x in z[f"{name}/params"])
        out.append(dict(name=name, A=z[f"{name}/A"], k=k, ell=ell, q=q, seed=seed, stream=stream, L=z[f"{name}/L"]))
    return out


def rpca_cases():
    """alm_rpca (rpca.hpp:95-169) with the CoR-UTV inner, outputs of the reference (make_golden.py rpca)."""
    z = np.load(os.path.join(HERE, "rpca_ref_cases.npz"))
    out = []
    for name in z["names"]:
        name = str(name)
        c = z[f"{name}/cfg"]
        cfg = dict(lambda_=float(c[0]), mu0=float(c[1]), rho=float(c[2]), mu_bar=float(c[3]), tol=float(c[4]),
                   max_iter=int(c[5]), corutv_ell=int(c[6]), corutv_q=int(c[7]), thresholding=int(c[8]))
        it, rank, sl0, conv, clamped = (int(x) for x in z[f"{name}/out"])
        case = dict(name=name, M=z[f"{name}/M"], L=z[f"{name}/L"], S=z[f"{name}/S"], residuals=z[f"{name}/residuals"],
                    cfg=cfg, iterations=it, rank_l=rank, s_l0=sl0, converged=bool(conv), ell_clamped=bool(clamped),
                    seed=2, stream=0)
        if f"{name}/S_true" in z.files:
            case["S_true"] = z[f"{name}/S_true"]
        out.append(case)
    return out
