"""Model check of the cross-GPU exchange protocol of dist.cu / steps.cu (peer mode), on CPU.

Each rank p, at iteration t: (1) publishes its partial, tagged t+1, into slot [t mod 2][p] of EVERY
rank's receive buffer; (2) waits until slot [t mod 2][r] of its OWN buffer carries tag t+1 for all r;
(3) reads them and sums in rank order.  The claim (dist.cu header): two parity slots suffice -- no
rank ever reads a slot already overwritten by iteration t+2, and the protocol never deadlocks.  Here
ranks are interleaved by random schedulers step by step (publish to one peer at a time, poll one slot
at a time), and every read is checked against what was published for that iteration.
"""
import random

import pytest


def run(P, T, seed):
    rng = random.Random(seed)
    buf = [[[(0, None) for _ in range(P)] for _ in range(2)] for _ in range(P)]  # [owner][slot][src]
    state = [{"t": 0, "phase": "pub", "i": 0, "got": []} for _ in range(P)]
    sums = [[] for _ in range(P)]
    value = lambda p, t: (p + 1) * 1000 + t  # what rank p publishes at iteration t
    steps = 0
    while any(s["t"] < T for s in state):
        steps += 1
        assert steps < 200 * P * P * T, "no progress (deadlock)"
        p = rng.randrange(P)
        s = state[p]
        t = s["t"]
        if t >= T:
            continue
        if s["phase"] == "pub":  # one remote store per step
            dst = s["i"]
            buf[dst][t % 2][p] = (t + 1, value(p, t))
            s["i"] += 1
            if s["i"] == P:
                s["phase"], s["i"], s["got"] = "poll", 0, []
        else:  # one poll per step; a slot is consumed when its tag matches
            r = s["i"]
            tag, v = buf[p][t % 2][r]
            assert tag <= t + 1, f"rank {p} slot overwritten by a later iteration (tag {tag} at t={t})"
            if tag == t + 1:
                assert v == value(r, t)
                s["got"].append(v)
                s["i"] += 1
                if s["i"] == P:
                    sums[p].append(sum(s["got"]))
                    s["t"], s["phase"], s["i"] = t + 1, "pub", 0
    # every rank saw the same totals, in the same order
    for p in range(1, P):
        assert sums[p] == sums[0]
    assert sums[0] == [sum(value(r, t) for r in range(P)) for t in range(T)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_two_slot_protocol(P):
    for seed in range(40):
        run(P, 12, seed)


def test_one_slot_would_fail():
    """The same protocol with ONE slot is not safe: some interleaving overwrites an unread value."""
    def run1(P, T, seed):
        rng = random.Random(seed)
        buf = [[(0, None) for _ in range(P)] for _ in range(P)]
        state = [{"t": 0, "phase": "pub", "i": 0} for _ in range(P)]
        for _ in range(100 * P * P * T):
            p = rng.randrange(P)
            s = state[p]
            t = s["t"]
            if t >= T:
                continue
            if s["phase"] == "pub":
                buf[s["i"]][p] = (t + 1, t)
                s["i"] += 1
                if s["i"] == P:
                    s["phase"], s["i"] = "poll", 0
            else:
                tag, _ = buf[p][s["i"]]
                if tag > t + 1:
                    return True  # overwritten before it was read
                if tag == t + 1:
                    s["i"] += 1
                    if s["i"] == P:
                        s["t"], s["phase"], s["i"] = t + 1, "pub", 0
        return False
    assert any(run1(2, 8, seed) for seed in range(200))
