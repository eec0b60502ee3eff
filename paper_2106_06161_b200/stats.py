"""GPU uniformity checks over batched shuffles -- the reference's statistical
tests (proj/include/bijshuf/stats.hpp) driven by the sm_100a batched kernel.

Samples follow BijectiveShuffleSampler (stats.hpp:314-324): draw b is
shuffle_indices(n, cfg with seed = cfg.seed + b), produced here by ONE
batched launch.  Because the permutations are bit-identical to the
reference's, every statistic equals the reference's for the same inputs.

    chi_squared_test  stats.hpp:247-276 (120 cells of S_5, 119 dof)
    mmd_test          stats.hpp:281-306 (Mallows kernel, normal / Hoeffding thresholds)
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass

from . import BijectionVariant, InvalidArgument, ShuffleConfig, shuffle_values_batched


class TestKind(enum.IntEnum):  # stats.hpp:232
    ChiSquared = 0
    MmdHoeffding = 1
    MmdNormal = 2


@dataclass
class TestReport:  # stats.hpp:234-241
    test_kind: TestKind
    statistic: float
    threshold: float
    alpha: float
    sample_size: int
    passed: bool


def sample_permutations(n: int, num_samples: int, cfg: ShuffleConfig, device="cuda"):
    """(num_samples, n) int64 CUDA tensor; row b = shuffle_indices(n, seed = cfg.seed + b)."""
    import torch
    dt = torch.int32 if n < 2**31 else torch.int64
    rows = torch.arange(n, dtype=dt, device=device).repeat(num_samples, 1)
    return shuffle_values_batched(rows, cfg).to(torch.int64)


def permutation_rank(perms):
    """Lehmer rank of each row (permutation.hpp:109-123), n <= 20."""
    import torch
    n = perms.shape[1]
    if n > 20:
        raise OverflowError("permutation_rank: n! overflows past n=20")
    rank = torch.zeros(perms.shape[0], dtype=torch.int64, device=perms.device)
    fact = math.factorial(n - 1) if n > 0 else 1
    for i in range(n):
        smaller_after = (perms[:, i + 1:] < perms[:, i:i + 1]).sum(dim=1)
        rank += smaller_after * fact
        if i + 1 < n:
            fact //= (n - 1 - i)
    return rank


def kendall_distance(a, b, chunk: int = 64):
    """Discordant pairs between rows a[i] and b[i] (permutation.hpp:93-105), on the GPU."""
    import torch
    n = a.shape[1]
    out = torch.empty(a.shape[0], dtype=torch.int64, device=a.device)
    for s in range(0, a.shape[0], chunk):
        aa, bb = a[s:s + chunk], b[s:s + chunk]
        pos = torch.empty_like(aa)
        pos.scatter_(1, aa, torch.arange(n, device=a.device).expand_as(aa))  # pos[sigma[k]] = k
        rel = torch.gather(bb, 1, pos)  # relabeled[r] = sigma'[position[r]]
        inv = (rel.unsqueeze(2) > rel.unsqueeze(1)).triu(diagonal=1).sum(dim=(1, 2))
        out[s:s + chunk] = inv
    return out


def chi2_quantile(p: float, k: int) -> float:  # stats.hpp:205-226
    from scipy.stats import chi2
    return float(chi2.ppf(p, k))


def chi_squared_test(num_samples: int, cfg: ShuffleConfig, alpha: float, device="cuda") -> TestReport:
    """stats.hpp:247-276 over GPU-batched length-5 shuffles."""
    import torch
    if num_samples < 12000:
        raise InvalidArgument("chi_squared_test: need >= 12000 samples")
    if not 0.0 < alpha < 1.0:
        raise InvalidArgument("chi_squared_test: alpha must be in (0, 1)")
    perms = sample_permutations(5, num_samples, cfg, device)
    counts = torch.bincount(permutation_rank(perms), minlength=120).double()
    expected = num_samples / 120.0
    stat = float(((counts - expected) ** 2 / expected).sum())
    thr = chi2_quantile(1.0 - alpha, 119)
    return TestReport(TestKind.ChiSquared, stat, thr, alpha, num_samples, stat < thr)


def _log1mexp(x: float) -> float:
    return math.log(-math.expm1(-x))


def mallows_expectation(n: int, lam: float) -> float:  # stats.hpp:41-53
    if n < 2 or lam < 0:
        raise InvalidArgument("mallows_expectation: bad arguments")
    if lam == 0:
        return 1.0
    unit = lam / (0.5 * n * (n - 1))
    s = 0.0
    for j in range(1, n + 1):
        s += _log1mexp(unit * j) - math.log(j) - _log1mexp(unit)
    return math.exp(s)


def mallows_variance(n: int, lam: float) -> float:  # stats.hpp:57-62
    mean = mallows_expectation(n, lam)
    v = mallows_expectation(n, 2 * lam) - mean * mean
    return max(v, 0.0)


def hoeffding_threshold(alpha: float, sample_size: int) -> float:  # stats.hpp:105-111
    return math.sqrt(math.log(2.0 / alpha) / sample_size)


def normal_threshold(alpha: float, n: int, lam: float, sample_size: int) -> float:  # stats.hpp:139-148
    from scipy.special import erfinv
    var_mmd = 2.0 * mallows_variance(n, lam) / sample_size
    return math.sqrt(2.0 * var_mmd) * float(erfinv(1.0 - alpha))


def mmd2_estimate(perms, lam: float) -> float:  # stats.hpp:88-101
    if perms.shape[0] == 0 or perms.shape[0] % 2:
        raise InvalidArgument("mmd2_estimate: sample count must be even and > 0")
    n = perms.shape[1]
    d = kendall_distance(perms[0::2], perms[1::2]).double()
    k = (-lam * d / (0.5 * n * (n - 1))).exp()
    mean_kernel = 2.0 * float(k.sum()) / perms.shape[0]
    return mean_kernel - mallows_expectation(n, lam)


def mmd_test(n: int, num_samples: int, cfg: ShuffleConfig, alpha: float, kind: TestKind, lam: float = 5.0,
             perms=None, device="cuda") -> TestReport:
    """stats.hpp:281-306; `perms` overrides the sampler (e.g. a point mass for the negative control)."""
    if kind not in (TestKind.MmdHoeffding, TestKind.MmdNormal):
        raise InvalidArgument("mmd_test: kind must be an MMD kind")
    if num_samples < 2 or num_samples % 2:
        raise InvalidArgument("mmd_test: num_samples must be even and >= 2")
    if perms is None:
        perms = sample_permutations(n, num_samples, cfg, device)
    stat = mmd2_estimate(perms, lam)
    thr = hoeffding_threshold(alpha, num_samples) if kind == TestKind.MmdHoeffding else \
        normal_threshold(alpha, n, lam, num_samples)
    return TestReport(kind, stat, thr, alpha, num_samples, abs(stat) < thr)


__all__ = ["TestKind", "TestReport", "sample_permutations", "permutation_rank", "kendall_distance",
           "chi_squared_test", "mmd_test", "mmd2_estimate", "mallows_expectation", "mallows_variance",
           "hoeffding_threshold", "normal_threshold", "chi2_quantile", "BijectionVariant"]
