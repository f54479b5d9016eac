"""Host model of the long-leaf Fisher-Yates rounds of `fy_leaf_warp`
(paper_2302_03317_b200/csrc/kernels_leaf.cu; Fisher-Yates: Fig. 1).

The kernel runs the steps i = m-1 .. 1 of `swap(A[i], A[j_i])` in rounds: the
32 lanes take the next 32 steps, mark their own position and then their
partner in a byte map, and the longest prefix of lanes none of whose marks was
overwritten runs at once (a flagged lane 0 runs alone).  Which of several
same-address stores of one warp instruction survives is unspecified by the PTX
ISA, so the model replays the rounds under three survivor policies (lowest
lane, highest lane, random) and checks each against the sequential loop.  No
oracle and no GPU code involved: this pins the round rule itself."""
import random

import pytest


def sequential(a, partners):
    a = list(a)
    for i in range(len(a) - 1, 0, -1):
        j = partners[i]
        a[i], a[j] = a[j], a[i]
    return a


def store_all(M, writes, policy, rng):
    """One warp store instruction: `writes` = [(lane, address)], the survivor
    per address chosen by `policy`."""
    by_addr = {}
    for lane, addr in writes:
        by_addr.setdefault(addr, []).append(lane)
    for addr, lanes in by_addr.items():
        if policy == "lowest":
            M[addr] = min(lanes)
        elif policy == "highest":
            M[addr] = max(lanes)
        else:
            M[addr] = rng.choice(lanes)


def rounds(a, partners, policy, seed=0):
    rng = random.Random(seed)
    a = list(a)
    m = len(a)
    M = [0xEE] * m  # stale content: the map is never cleared
    top = m - 1
    nrounds = 0
    while top >= 1:
        lanes = [(l, top - l) for l in range(32) if top - l >= 1]
        j = {l: partners[i] for l, i in lanes}
        va = {l: a[i] for l, i in lanes}
        vb = {l: a[j[l]] for l, _ in lanes}
        store_all(M, [(l, i) for l, i in lanes], policy, rng)      # own positions (distinct)
        store_all(M, [(l, j[l]) for l, _ in lanes], policy, rng)   # partners
        flagged = [l for l, i in lanes if M[j[l]] != l or M[i] != l]
        c = max(min(flagged), 1) if flagged else min(32, top)
        for l, i in lanes:
            if l < c:
                a[i] = vb[l]
                a[j[l]] = va[l]
        top -= c
        nrounds += 1
        assert nrounds <= m  # progress
    return a, nrounds


@pytest.mark.parametrize("policy", ["lowest", "highest", "random"])
@pytest.mark.parametrize("m", [2, 3, 31, 32, 33, 64, 100, 513, 2048])
def test_rounds_equal_sequential_fisher_yates(policy, m):
    rng = random.Random(m * 7919 + len(policy))
    for trial in range(20 if m <= 100 else 4):
        partners = [0] + [rng.randrange(i + 1) for i in range(1, m)]
        a = list(range(m))
        got, _ = rounds(a, partners, policy, seed=trial)
        assert got == sequential(a, partners)


@pytest.mark.parametrize("policy", ["lowest", "highest", "random"])
def test_rounds_adversarial_partners(policy):
    """All steps share one partner; every partner is the next lane's position;
    self-swaps only; lane 0 shares its partner with every other lane."""
    m = 200
    cases = [
        [0] * m,                                       # one partner for all
        [0] + [i - 1 for i in range(1, m)],            # partner = the next step's position
        list(range(m)),                                # self-swaps
        [0] + [min(i, 5) for i in range(1, m)],        # a few hot partners
        [0] + [(i // 2) for i in range(1, m)],
    ]
    for partners in cases:
        a = list(range(m))
        got, _ = rounds(a, partners, policy, seed=1)
        assert got == sequential(a, partners)


def test_round_count_on_uniform_partners():
    """~sqrt(i) steps per round at small i, 32 at large i: a 2048-element leaf
    takes on the order of a hundred rounds (leaf kernel)."""
    rng = random.Random(5)
    m = 2048
    partners = [0] + [rng.randrange(i + 1) for i in range(1, m)]
    _, n = rounds(list(range(m)), partners, "lowest")
    assert 64 <= n <= 200
