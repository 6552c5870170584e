"""The bulge-chasing dependency rule of the CUDA chase (b2t.cu chase_kernel): sweep s task t
may run once sweep s-1 finished tasks 0..t+1, because it shares exactly one entry with s-1's
task t+2 -- A(r', col'), the entry that task's Householder overwrites with beta first -- and
nothing with later tasks of s-1 or with tasks >= t+3 of s-2.  Checked on exact access sets,
and numerically: an adversarial interleaving allowed by the rule reproduces the sequential
chase exactly.  (Host-side model of the schedule; the task geometry follows PAPER.md:446-462
as implemented in b2t.cu.)"""
import numpy as np
import pytest


def ntask(n, b, s):
    return 1 + (n - 3 - s) // b


def geom(n, b, s, t):
    if t == 0:
        col, r, L = s, s + 1, min(b, n - 1 - s)
    else:
        col = s + 1 + (t - 1) * b
        r = col + b
        L = min(b, n - r)
    return col, r, L, min(n, r + L + b)


def access(n, b, s, t):
    col, r, L, e = geom(n, b, s, t)
    S = {(i, c) for c in range(col, r) for i in range(r, r + L)}
    S |= {(i, c) for c in range(r, r + L) for i in range(c + 1, e)}
    return S


@pytest.mark.parametrize("n,b", [(20, 2), (33, 3), (50, 4), (71, 8)])
def test_access_sets(n, b):
    for s in range(1, n - 2):
        for t in range(ntask(n, b, s)):
            A = access(n, b, s, t)
            e = geom(n, b, s, t)[3]
            for tp in range(t + 2, ntask(n, b, s - 1)):
                inter = A & access(n, b, s - 1, tp)
                if tp == t + 2:
                    colp, rp = geom(n, b, s - 1, tp)[:2]
                    assert inter == ({(rp, colp)} if rp < e else set())
                else:
                    assert not inter
            if s >= 2:
                for tp in range(t + 3, ntask(n, b, s - 2)):
                    assert not (A & access(n, b, s - 2, tp))


def _larfg(x):
    v = np.zeros_like(x)
    v[0] = 1.0
    xn = np.linalg.norm(x[1:])
    if xn == 0.0:
        return v, 0.0, x[0]
    beta = -np.copysign(np.hypot(x[0], xn), x[0])
    v[1:] = x[1:] / (x[0] - beta)
    return v, (beta - x[0]) / beta, beta


def _run(n, b, order, seed=1):
    rng = np.random.default_rng(seed)
    M = np.tril(rng.uniform(-1, 1, (n, n)), -1)
    M[np.subtract.outer(np.arange(n), np.arange(n)) > b] = 0.0
    pend = {}
    for kind, s, t in order:
        col, r, L, e = geom(n, b, s, t)
        if kind == "h":   # Householder: column col -> beta e1
            v, tau, beta = _larfg(M[r:r + L, col].copy())
            M[r:r + L, col] = 0.0
            M[r, col] = beta
            pend[(s, t)] = (v, tau)
            continue
        v, tau = pend.pop((s, t))
        S = np.tril(M, -1)
        S = S - S.T
        rs = slice(r, r + L)
        S[rs, col + 1:r] -= tau * np.outer(v, v @ S[rs, col + 1:r])
        S[col + 1:r, rs] = -S[rs, col + 1:r].T
        D = S[rs, rs]
        w = tau * (D @ v)
        S[rs, rs] = D + np.outer(v, w) - np.outer(w, v)
        E = S[r + L:e, rs]
        S[r + L:e, rs] = E - np.outer(tau * (E @ v), v)
        M = np.tril(S, -1)
    return -np.diag(M, -1)


def _adversarial(n, b):
    """Greedy order that always advances the highest sweep the rule allows."""
    done, nxt, inh, order = {}, {s: 0 for s in range(n - 2)}, set(), []
    while True:
        cands = []
        for s in range(n - 2):
            t = nxt[s]
            if t >= ntask(n, b, s):
                continue
            if (s, t) in inh:
                cands.append(("u", s, t))
                continue
            if s > 0:
                tp = ntask(n, b, s - 1)
                e = geom(n, b, s, t)[3]
                if t + 2 < tp and geom(n, b, s - 1, t + 2)[1] < e:
                    # needs tasks 0..t+1 done and the Householder (beta) of task t+2
                    if not (done.get(s - 1, 0) >= t + 2 and ((s - 1, t + 2) in inh or done.get(s - 1, 0) >= t + 3)):
                        continue
                elif done.get(s - 1, 0) < min(t + 2, tp):
                    continue
            cands.append(("h", s, t))
        if not cands:
            return order
        k, s, t = max(cands, key=lambda c: c[1])
        order.append((k, s, t))
        if k == "h":
            inh.add((s, t))
        else:
            inh.discard((s, t))
            done[s] = t + 1
            nxt[s] = t + 1


@pytest.mark.parametrize("n,b", [(40, 4), (64, 8)])
def test_interleaving_reproduces_sequential(n, b):
    seq = [(k, s, t) for s in range(n - 2) for t in range(ntask(n, b, s)) for k in "hu"]
    adv = _adversarial(n, b)
    assert sorted(adv) == sorted(seq)
    pos = {x: i for i, x in enumerate(adv)}
    reordered = sum(1 for (k, s, t) in adv if k == "u" and s > 0 and ("u", s - 1, t + 2) in pos
                    and pos[("u", s, t)] < pos[("u", s - 1, t + 2)])
    assert reordered > 0, "the interleaving must actually exercise the relaxed rule"
    np.testing.assert_array_equal(_run(n, b, adv), _run(n, b, seq))
