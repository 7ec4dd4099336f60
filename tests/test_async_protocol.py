"""CPU models of the termination protocols of the asynchronous kernels
(no barrier between relaxations):

* "grid" -- the two-wave S/R protocol of both asynchronous kernels
  (csrc/gasync.cu: S per warp, R per CTA, in global memory; csrc/cluster.cu
  ASYNC: S and R per CTA in shared memory, read through DSMEM): S counts
  marks (counted BEFORE the bit is set, minus marks that hit an already-set
  bit), R taken vertices whose relaxations finished; an idle CTA 0 sums
  every R, then every S, and stops everyone when the sums are equal (the
  model keeps one S per CTA: finer counters only spread the same sums);
* "cluster" -- one pending counter (+k before marking, -dups after, -F
  after finishing F taken vertices; idle CTAs stop when it reads 0): the
  cluster kernel's protocol until round 2 session 3, kept as a checked
  alternative (every marking warp waiting on one shared word made the
  kernel 7 % slower once the wait was enforced).

Every shared-memory access of the protocol is one step of a generator; a
seeded random scheduler interleaves the "CTAs" one step at a time (the
adversarial interleavings the hardware may produce).  Checked: whenever a
stop is decided, no vertex is marked and none is being processed (no false
termination), and the final arrivals equal the serial CSA oracle.  A
deliberately broken variant (S counted AFTER the bit is set) must be caught
by the same check for some interleaving -- the test has teeth.
Speculative counting (``spec``, the kernels since round 2 session 3): a
warp counts every lane that TRIES to lower e[v] before its atomicMins (the
count and the atomicMins share one round trip), sets the bits of the
vertices it lowered, then subtracts the tries that lowered nothing and the
marks that hit a set bit.

The relaxation itself is a test-side model on the raw connections (the CUDA
relaxation is covered by the GPU parity tests); what is tested is the
take / mark / count / detect protocol.
"""
import random

import numpy as np

import oracle
import synth

INF = oracle.INF


class _World:
    def __init__(self, tt, s, t_s, P):
        self.n, self.P = tt.num_vertices, P
        self.out = [[] for _ in range(self.n)]
        for u, v, d, l in zip(tt.u.tolist(), tt.v.tolist(), tt.dep.tolist(), tt.dur.tolist()):
            self.out[u].append((v, d, l))
        self.e = [INF] * self.n
        self.bits = [False] * self.n
        self.e[s] = t_s
        self.bits[s] = True
        self.S = [0] * P
        self.R = [0] * P
        self.pend = 1                 # cluster protocol: the source is pending
        self.S[s % P] = 1             # grid protocol: the source's mark, counted by its owner
        self.done = False
        self.processing = [0] * P     # vertices taken and not yet finished (for the check)

    def owner(self, v):
        return v % self.P

    def pending_work(self):
        return any(self.bits) or any(self.processing)


def _cta(wd, me, protocol, broken, log, spec=False):
    """One CTA: a generator, one shared-memory access per step."""
    while True:
        # take every marked vertex this CTA owns (atomicExch per vertex)
        taken = []
        for v in range(me, wd.n, wd.P):
            yield
            if wd.bits[v]:
                wd.bits[v] = False
                taken.append(v)
        wd.processing[me] = len(taken)
        if not taken:
            # idle: detect (grid: CTA 0) / poll
            if protocol == "grid":
                if me == 0:
                    ra = 0
                    for r in range(wd.P):
                        yield
                        ra += wd.R[r]
                    sb = 0
                    for r in range(wd.P):
                        yield
                        sb += wd.S[r]
                    if ra == sb:
                        log.append(wd.pending_work())  # a stop decided while work is pending is a bug
                        wd.done = True
                yield
                if wd.done:
                    return
            else:
                yield
                if wd.pend == 0:
                    log.append(wd.pending_work())
                    return
            continue
        late = 0  # broken variant: marks counted only when the iteration ends
        for u in taken:
            yield
            eu = wd.e[u]
            lowered = []
            if spec:
                tries = []
                for v, d, l in wd.out[u]:
                    yield
                    if d >= eu and d + l < wd.e[v]:  # e[v] read: this lane will try
                        tries.append((v, d + l))
                if tries:
                    yield  # the returning count, before any atomicMin or bit
                    if protocol == "grid":
                        wd.S[me] += len(tries)
                    else:
                        wd.pend += len(tries)
                    for v, c in tries:
                        yield
                        if c < wd.e[v]:  # atomicMin
                            wd.e[v] = c
                            lowered.append(v)
                    dups = 0
                    for v in lowered:
                        yield
                        if wd.bits[v]:
                            dups += 1
                        wd.bits[v] = True
                    yield  # un-count the tries that lowered nothing and the duplicates
                    if protocol == "grid":
                        wd.S[me] -= len(tries) - len(lowered) + dups
                    else:
                        wd.pend -= len(tries) - len(lowered) + dups
                lowered = []
            for v, d, l in ([] if spec else wd.out[u]):
                if d >= eu and d + l < wd.e[v]:
                    yield
                    if d + l < wd.e[v]:  # atomicMin
                        wd.e[v] = d + l
                        lowered.append(v)
            # mark them (a warp's marks: count first, then set, then un-count duplicates)
            if lowered:
                if not broken:
                    yield
                    if protocol == "grid":
                        wd.S[me] += len(lowered)
                    else:
                        wd.pend += len(lowered)
                dups = 0
                for v in lowered:
                    yield
                    if wd.bits[v]:
                        dups += 1
                    wd.bits[v] = True
                if broken:
                    late += len(lowered) - dups
                else:
                    yield
                    if protocol == "grid":
                        wd.S[me] -= dups
                    else:
                        wd.pend -= dups
        if broken:  # "publish the counters at the end of the iteration": too late
            yield
            if protocol == "grid":
                wd.S[me] += late
            else:
                wd.pend += late
        # the taken vertices are done (after every mark they made was counted)
        yield
        if protocol == "grid":
            wd.R[me] += len(taken)
        else:
            wd.pend -= len(taken)
        wd.processing[me] = 0


def _run(tt, s, t_s, P, protocol, broken, seed, max_steps=2_000_000, spec=False):
    wd = _World(tt, s, t_s, P)
    log = []
    ctas = [_cta(wd, me, protocol, broken, log, spec) for me in range(P)]
    live = list(range(P))
    rng = random.Random(seed)
    steps = 0
    while live and steps < max_steps:
        i = rng.choice(live)  # a burst of 1..24 steps of one CTA: long starvation windows for the others
        for _ in range(rng.randint(1, 24)):
            try:
                next(ctas[i])
            except StopIteration:
                live.remove(i)
                break
            steps += 1
    assert steps < max_steps, "protocol model did not terminate"
    return wd, log


def _instances():
    for seed in range(40):
        tt = synth.random_small(seed, nmax=24, cmax=160)
        rng = np.random.default_rng(seed)
        yield seed, tt, int(rng.integers(tt.num_vertices)), int(rng.integers(0, 2 * 86400))


def test_async_termination_protocols_match_oracle():
    for seed, tt, s, t_s in _instances():
        want = oracle.CSA(tt.num_vertices, *tt.arrays()).query(s, t_s)
        for protocol in ("grid", "cluster"):
            for P in (1, 2, 3, 5):
                for spec in (False, True):
                    wd, log = _run(tt, s, t_s, P, protocol, broken=False, seed=seed * 31 + P, spec=spec)
                    tag = f"{protocol} P={P} spec={spec} seed={seed}"
                    assert log and not any(log), f"{tag}: stop decided with work pending"
                    assert not wd.pending_work()
                    assert np.array_equal(np.array(wd.e, dtype=np.uint32), want), tag


def test_counting_after_marking_is_caught():
    """Negative control: counting the marks only when the iteration ends
    (after their bits are visible) lets the detector stop while an owner
    still has work -- some interleaving of these instances must expose it
    (a stop with work pending, or a wrong row)."""
    caught = False
    for seed, tt, s, t_s in _instances():
        want = oracle.CSA(tt.num_vertices, *tt.arrays()).query(s, t_s)
        for trial in range(40):
            wd, log = _run(tt, s, t_s, 2 + trial % 2, "grid", broken=True, seed=seed * 1000 + trial)
            if any(log) or not np.array_equal(np.array(wd.e, dtype=np.uint32), want):
                caught = True
                break
        if caught:
            break
    assert caught, "the broken counting order was never caught: the model has no teeth"
