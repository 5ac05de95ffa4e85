"""Algorithm 1 (covariance splitting) through bsf_run_alg1
against a two-stage oracle: the oracle's direct-sum filter applied with the
isotropic covariance sigma_b^2 I to every pixel, then with C - sigma_b^2 I to
that float64 image (Proposition 2: the composition is one
space-variant filter)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import make_plan, max_rel
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu


def _bound9(cov, policy, clamp=1):
    """Eq. (9) per pixel with the basis each pixel uses and
    the clamped covariance (R21); e(phi) as rho_B."""
    sx, sy, th = (cov[i].astype(np.float64) for i in range(3))
    swap = sx < sy
    phi = np.where(swap, th + math.pi / 2, th) % math.pi
    l1 = np.maximum(sx, sy) ** 2
    l2 = np.minimum(sx, sy) ** 2
    s2, c2 = np.abs(np.sin(2 * phi)), np.abs(np.cos(2 * phi))
    eT = 1.0 / (s2 + c2)
    with np.errstate(divide="ignore"):
        eP = np.minimum(np.where(c2 > 0, 0.6 / c2, np.inf), np.where(s2 > 0, 0.8 / s2, np.inf))
    if policy == 2:
        theta_prime = (sx != sy) & (eP > eT)
    else:
        theta_prime = np.full(sx.shape, policy == 1)
    eb = np.where(theta_prime, eP, eT)
    rb = np.where(eb < 1, (1 + eb) / np.maximum(1 - eb, 1e-300), np.inf)
    rho = l1 / l2
    cl = clamp & (eb < 1) & (sx != sy) & (rho > 0.95 * rb)
    T = l1 + l2
    lim = 0.95 * rb
    with np.errstate(invalid="ignore"):
        e = np.where(cl, (lim - 1) / (lim + 1), 0.0)
    l1 = np.where(cl, 0.5 * T * (1 + e), l1)
    l2 = np.where(cl, 0.5 * T * (1 - e), l2)
    return 0.5 * (l1 + l2 - (l1 - l2) / np.minimum(eb, 1.0))


@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("r", [1, 2])
def test_alg1_matches_two_stage_oracle(policy, r):
    H, W = 34, 40
    w, img, cov = _small_smooth(H, W, 3.5, seed=21)
    plan = make_plan(w, policy=policy, order=r, anchor=bsf.BSF_ANCHOR_TILE)
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    sig = plan.run_alg1(img[None].cuda().contiguous(), cov.cuda().contiguous(), out)
    torch.cuda.synchronize()
    c = cov.numpy()
    # sigma_b^2 = half the smallest bound (9) over the field
    s2 = 0.5 * float(_bound9(c, policy).min())
    assert abs(sig[0] - s2) <= 1e-12 * s2, (sig[0], s2)
    s = math.sqrt(sig[0])
    ys, xs = np.mgrid[0:H, 0:W]
    xs, ys = xs.ravel(), ys.ravel()
    g, *_ = O.filter_points(img.numpy(), xs, ys, s, s, 0.0, policy=policy, r=r)
    g = g.reshape(H, W)
    sx = np.sqrt(np.maximum(c[0].astype(np.float64) ** 2 - sig[0], 0.0))[ys, xs]
    sy = np.sqrt(np.maximum(c[1].astype(np.float64) ** 2 - sig[0], 0.0))[ys, xs]
    ref, *_ = O.filter_points(g, xs, ys, sx, sy, c[2][ys, xs].astype(np.float64), policy=policy, r=r)
    got = out[0].cpu().numpy().ravel()
    assert max_rel(got, ref) <= 1e-9
    assert plan.stats()["flags"] == 0


def test_alg1_batch_sigma_per_field():
    """One sigma_b per covariance field of a batch (channels share it)."""
    w = synth.workload(1, width=36, height=30, batch=2, channels=2)
    imgs = torch.stack([synth.make_image(w, frame=b, channel=c) for b in range(2) for c in range(2)])
    covs = torch.stack([synth.make_cov(w) for _ in range(2)])
    covs[1, 0] *= 2.0
    covs[1, 1] *= 1.5
    plan = make_plan(w, anchor=bsf.BSF_ANCHOR_TILE)
    out = torch.empty((4, 30, 36), dtype=torch.float64, device="cuda")
    sig = plan.run_alg1(imgs.cuda().contiguous(), covs.cuda().contiguous(), out)
    torch.cuda.synchronize()
    for b in range(2):
        s2 = 0.5 * float(_bound9(covs[b].numpy(), 2).min())
        assert abs(sig[b] - s2) <= 1e-12 * s2
    assert sig[1] > sig[0]
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("policy", [0, 2])
def test_alg1_closer_to_the_gaussian(policy):
    """The paper's claim (Table 2): splitting the covariance
    improves the Gaussian approximation.  Impulse response of the plain order-1
    filter and of Algorithm 1 (same target covariance C, constant field) vs the
    sampled Gaussian of covariance C: Algorithm 1 has the smaller L2 error."""
    H = W = 49
    w = synth.workload(2, width=W, height=H, max_sigma=6.0)
    img = torch.zeros((H, W), dtype=torch.float32)
    img[H // 2, W // 2] = 1.0
    smaj, rho, th = 4.5, 2.0, math.radians(30.0)
    cov = torch.tensor([smaj, smaj / math.sqrt(rho), th], dtype=torch.float32)[:, None, None].expand(3, H, W)
    cov = cov.contiguous()
    plan = make_plan(w, policy=policy, order=1, anchor=bsf.BSF_ANCHOR_TILE)
    plain = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run(img[None].cuda(), cov.cuda(), plain)
    alg1 = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run_alg1(img[None].cuda(), cov.cuda(), alg1)
    torch.cuda.synchronize()
    # sampled Gaussian of covariance C = R diag(sx^2, sy^2) R^T (impulse response)
    sx, sy = smaj, smaj / math.sqrt(rho)
    c, s = math.cos(th), math.sin(th)
    C = np.array([[sx * sx * c * c + sy * sy * s * s, (sx * sx - sy * sy) * s * c],
                  [(sx * sx - sy * sy) * s * c, sx * sx * s * s + sy * sy * c * c]])
    Ci = np.linalg.inv(C)
    yy, xx = np.mgrid[0:H, 0:W]
    d = np.stack([xx - W // 2, yy - H // 2], -1).astype(np.float64)
    gauss = np.exp(-0.5 * np.einsum("...i,ij,...j->...", d, Ci, d)) / (2 * math.pi * math.sqrt(np.linalg.det(C)))
    err = lambda k: float(np.linalg.norm(k - gauss) / np.linalg.norm(gauss))
    e_plain, e_alg1 = err(plain[0].cpu().numpy()), err(alg1[0].cpu().numpy())
    assert e_alg1 < 0.75 * e_plain, (e_plain, e_alg1)


def test_split_two_passes_is_algorithm1():
    """bsf_run_split with n = 2 is Algorithm 1, bit for bit."""
    H, W = 34, 40
    w, img, cov = _small_smooth(H, W, 3.5, seed=22)
    plan = make_plan(w, policy=2, order=1, anchor=bsf.BSF_ANCHOR_TILE)
    a = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    s1 = plan.run_alg1(img[None].cuda().contiguous(), cov.cuda().contiguous(), a)
    s2 = plan.run_split(img[None].cuda().contiguous(), cov.cuda().contiguous(), b, 2)
    torch.cuda.synchronize()
    assert s1[0] == s2[0] and torch.equal(a, b)


@pytest.mark.parametrize("policy,r,n", [(0, 1, 3), (2, 1, 4), (2, 2, 3)])
def test_split_matches_multi_stage_oracle(policy, r, n):
    """n - 1 isotropic passes of (B/n) I then C - ((n-1) B/n) I (R22),
    against the oracle applied stage by stage to every pixel (float64
    intermediates; Proposition 2 composes them)."""
    H, W = 30, 34
    w, img, cov = _small_smooth(H, W, 3.5, seed=23)
    plan = make_plan(w, policy=policy, order=r, anchor=bsf.BSF_ANCHOR_TILE)
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    sig = plan.run_split(img[None].cuda().contiguous(), cov.cuda().contiguous(), out, n)
    torch.cuda.synchronize()
    c = cov.numpy()
    bound = float(_bound9(c, policy).min())
    assert abs(2.0 * sig[0] - bound) <= 1e-12 * bound
    ys, xs = np.mgrid[0:H, 0:W]
    xs, ys = xs.ravel(), ys.ravel()
    g = img.numpy()
    s = math.sqrt(2.0 * sig[0] / n)
    for _ in range(n - 1):
        g, *_ = O.filter_points(g, xs, ys, s, s, 0.0, policy=policy, r=r)
        g = g.reshape(H, W)
    t = 2.0 * sig[0] * (n - 1) / n
    sx = np.sqrt(np.maximum(c[0].astype(np.float64) ** 2 - t, 0.0))[ys, xs]
    sy = np.sqrt(np.maximum(c[1].astype(np.float64) ** 2 - t, 0.0))[ys, xs]
    ref, *_ = O.filter_points(g, xs, ys, sx, sy, c[2][ys, xs].astype(np.float64), policy=policy, r=r)
    got = out[0].cpu().numpy().ravel()
    assert max_rel(got, ref) <= 1e-9
    assert plan.stats()["flags"] == 0


def _impulse_errors(fracs, smaj=5.0, rho=3.0, theta=math.pi / 4, policy=2):
    """L2 error (relative) of impulse responses against the sampled Gaussian of
    the same covariance: the plain order-1 filter, then the two-pass split with
    isotropic share `frac` of the bound (9) for each frac."""
    H = W = 61
    w = synth.workload(2, width=W, height=H, max_sigma=smaj + 1.0)
    img = torch.zeros((H, W), dtype=torch.float32)
    img[H // 2, W // 2] = 1.0
    cov = torch.tensor([smaj, smaj / math.sqrt(rho), theta], dtype=torch.float32)[:, None, None].expand(3, H, W)
    cov = cov.contiguous().cuda()
    plan = make_plan(w, policy=policy, order=1, anchor=bsf.BSF_ANCHOR_TILE)
    sx, sy = smaj, smaj / math.sqrt(rho)
    c, s = math.cos(theta), math.sin(theta)
    C = np.array([[sx * sx * c * c + sy * sy * s * s, (sx * sx - sy * sy) * s * c],
                  [(sx * sx - sy * sy) * s * c, sx * sx * s * s + sy * sy * c * c]])
    Ci = np.linalg.inv(C)
    yy, xx = np.mgrid[0:H, 0:W]
    d = np.stack([xx - W // 2, yy - H // 2], -1).astype(np.float64)
    gauss = np.exp(-0.5 * np.einsum("...i,ij,...j->...", d, Ci, d)) / (2 * math.pi * math.sqrt(np.linalg.det(C)))
    err = lambda k: float(np.linalg.norm(k - gauss) / np.linalg.norm(gauss))
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run(img[None].cuda(), cov, out)
    torch.cuda.synchronize()
    e0 = err(out[0].cpu().numpy())
    es = []
    for fr in fracs:
        plan.run_split(img[None].cuda(), cov, out, 2, fr)
        torch.cuda.synchronize()
        es.append(err(out[0].cpu().numpy()))
    return e0, es


def test_table3_fraction_sweep_trend():
    """Table 3: the improvement of Algorithm 1 over the
    plain filter for the Gaussian (s = 5, rho = 3, theta = pi/4) as the
    isotropic share of the bound (9) sweeps 10..80 %.  The paper's values come
    from a continuous-domain protocol (not reproduced); on the
    sampled impulse response the trend it reports holds: small shares help
    little, the improvement rises to ~50 % and stays within a few points of
    its maximum beyond."""
    fracs = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8]
    e0, es = _impulse_errors(fracs)
    imp = [1.0 - e / e0 for e in es]
    print("table 3 (sampled):", " ".join("%d%%:%.1f" % (100 * f, 100 * i) for f, i in zip(fracs, imp)))
    assert imp[0] < imp[4], imp
    assert all(imp[k] <= imp[k + 1] + 1e-3 for k in range(4)), imp  # rising up to 50 %
    assert imp[4] >= max(imp) - 0.05, imp  # 50 % within 5 points of the best


def test_table2_anisotropic_columns_improve():
    """Table 2, anisotropic columns (s, rho, theta) on the
    sampled impulse response (the paper's continuous-domain protocol is not
    reproduced: DESIGN.md): Algorithm 1 lowers the L2 error against the
    Gaussian in every case of size s = 5, as the paper reports (12.7-26.7 %).
    The (1, 4, 0) column is left out: with sigma_minor = 0.5 px the sampling
    between the two passes dominates the sampled response (plain 20 %, two
    passes 59 %), which the continuous-domain protocol does not see."""
    cases = [(5.0, 4.0, 0.0), (5.0, 3.0, math.pi / 8), (5.0, 8.0, math.pi / 3), (5.0, 5.0, math.pi / 2)]
    rows = []
    for s, rho, th in cases:
        e0, (e1,) = _impulse_errors([0.5], smaj=s, rho=rho, theta=th)
        rows.append((s, rho, th, e0, e1))
        assert e1 < e0, (s, rho, th, e0, e1)
    print("table 2 (sampled):", "; ".join("(%g,%g,%.3f) %.1f%% -> %.1f%%" % (s, r, t, 100 * a, 100 * b)
                                         for s, r, t, a, b in rows))
