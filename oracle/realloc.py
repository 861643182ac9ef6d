"""Oracle: lightweight sample reallocation policy (test infrastructure only).

PAPER.md section 6.1:
  * instance throughput "exhibits a roofline phenomenon"; the turning point is the
    *threshold* (P:268). Reading Z13: the smallest profiled count at which the
    marginal gain per added sample (backward difference) drops below 10% of the first
    segment's gain; linear profile -> largest count.
  * objective Eq. 6: maximise sum_j (d_next - d_cur) s.t. sources stay >= thr,
    destinations stay <= thr, every instance migrates at most once.
  * greedy: sort by load; repeatedly pair the instances with the largest difference
    (most-loaded source, least-loaded destination); move min(s_cur - thr, thr - d_cur)
    samples; prefer shorter sequences, then lower average accepted tokens (ties: gid).
  * decisions every `cooldown` steps, triggered only if the inefficiency is present.
"""
from __future__ import annotations


def knee_threshold(profile, frac=0.10):
    counts = [c for c, _ in profile]
    tput = [t for _, t in profile]
    if len(profile) < 3:
        raise ValueError("need >= 3 profile points")
    g0 = (tput[1] - tput[0]) / (counts[1] - counts[0])
    if g0 <= 0:
        return counts[0]
    for i in range(1, len(profile)):
        g = (tput[i] - tput[i - 1]) / (counts[i] - counts[i - 1])
        if g < frac * g0:
            return counts[i]
    return counts[-1]


def plan_reallocation(loads, thr):
    """loads: per-instance sample counts. Returns a list of (src, dst, count)."""
    srcs = sorted([i for i, x in enumerate(loads) if x > thr], key=lambda i: (-loads[i], i))
    dsts = sorted([i for i, x in enumerate(loads) if x < thr], key=lambda i: (loads[i], i))
    plan = []
    for s, d in zip(srcs, dsts):
        k = min(loads[s] - thr, thr - loads[d])
        if k <= 0:
            break
        plan.append((s, d, k))
    return plan


def choose_samples(samples, k):
    """samples: list of (gid, seq_len, avg_accepted). Shorter sequence first, then lower
    average accepted tokens, then lower gid. Returns the k chosen gids."""
    return [s[0] for s in sorted(samples, key=lambda s: (s[1], s[2], s[0]))[:k]]


def should_trigger(loads, thr, steps_since_last, cooldown=32):
    return (steps_since_last >= cooldown and any(x < thr for x in loads)
            and any(x > thr for x in loads))


def apply_plan(loads, plan):
    out = list(loads)
    for s, d, k in plan:
        out[s] -= k
        out[d] += k
    return out
