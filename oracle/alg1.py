"""TEST INFRASTRUCTURE ONLY -- a tiny pure-Python model of the paper's Algorithm 1
(PAPER.md P:72-119), written step by step in the paper's order and notation, for small
inputs.  It pins Table II, the S/L/R sets of the worked example
and the "calculations" arithmetic.  The parity authority is the plain
sequential walk (oracle.c); this model is checked against it by the partition-invariance
tests.

Readings (DESIGN.md / SURVEY.md §8(c)):
  C1  L uses the PREVIOUS chunk's last character ("last character of T_{p-1}"),
      not Alg. 1's garbled ``pi_input.back()``.
  C3  hits count destinations in F; the start state is not counted.
  C4  one hit counter per route (Alg. 1's single ``found`` would over-count when |R| > 1).
  C5  the join keys routes by start state: result(q) = right(left.end(q)).
  C6  Table II's last row is P_3 ("P_4" is a typo); under R = S n L it has R_3 = L(e) = {0,7}.
  C7  chunk i = T[i*floor(n/p) : ...], remainder to the last chunk; p clamped to [1, n].
  C9  DEAD ends a route: end = DEAD, hits so far; an arriving state outside R dies.
"""
from __future__ import annotations

from dataclasses import dataclass, field

DEAD = -1


@dataclass
class Route:                  # one r in R: Alg. 1 lines 16-25
    start: int
    visited: list = field(default_factory=list)   # Rr: one state per consumed char
    hits: int = 0

    @property
    def end(self) -> int:
        if self.visited and self.visited[-1] == DEAD:
            return DEAD
        return self.visited[-1] if self.visited else self.start


def delta(Tt, q, c):
    v = int(Tt[q][c])
    return DEAD if v in (0xFFFF, 0xFFFFFFFF, DEAD) else v


def chunk_input(T, p):
    """Alg. 1 lines 3-4: start_position = i * (T.length / p), remainder to last."""
    n = len(T)
    p = max(1, min(p, n)) if n else 1
    w = n // p if n else 0
    return [T[i * w:(i + 1) * w] if i < p - 1 else T[i * w:] for i in range(p)]


def S_set(Tt, first_char):
    """Alg. 1 lines 5-9: states with a transition on the chunk's first char."""
    return {q for q in range(len(Tt)) if delta(Tt, q, first_char) != DEAD}


def L_set(Tt, prev_last_char):
    """Alg. 1 lines 10-14 with reading C1: destinations on the previous
    chunk's last char."""
    return {delta(Tt, q, prev_last_char) for q in range(len(Tt))} - {DEAD}


def run_route(Tt, F, r, chunk) -> Route:
    """Alg. 1 lines 16-25: for char in chunk: if Tt[r][char] in F: found++;
    Rr[i] = r = Tt[r][char]."""
    route = Route(r)
    for ch in chunk:
        nxt = delta(Tt, r, ch)
        if nxt == DEAD:
            route.visited.append(DEAD)
            break
        if nxt in F:
            route.hits += 1
        route.visited.append(nxt)
        r = nxt
    return route


@dataclass
class ParemRun:
    chunks: list
    R: list                 # R_i per chunk (sorted lists)
    routes: list            # dict start -> Route per chunk
    final_state: int
    accepted: bool
    match_count: int

    @property
    def calculations(self) -> int:
        """Raw route count sum_i |R_i|."""
        return sum(len(r) for r in self.R)

    @property
    def distinct_after_first(self) -> int:
        """sum_i |{delta(r, first char of chunk i) : r in R_i}| -- the count under which the
        worked example gives the paper's "five calculations" (reading C6)."""
        tot = 0
        for R_i, routes in zip(self.R, self.routes):
            tot += len({routes[r].visited[0] if routes[r].visited else r for r in R_i})
        return tot


def run_parem(Tt, q0, F, T, p, enum=False) -> ParemRun:
    """Algorithm 1 followed by the barrier and the join.
    ``enum=True`` gives the General Enumeration Approach (every chunk i >= 1 starts
    from all of Q)."""
    F = set(F)
    chunks = chunk_input(T, p)
    Rs, routes = [], []
    for i, chunk in enumerate(chunks):
        if i == 0:
            R = {q0}                                  # "already knows ... q0"
        elif enum:
            R = set(range(len(Tt)))
        else:
            if not chunk:
                R = set()
            else:
                S = S_set(Tt, chunk[0])
                L = L_set(Tt, chunks[i - 1][-1])
                R = S & L                             # line 15
        Rs.append(sorted(R))
        routes.append({r: run_route(Tt, F, r, chunk) for r in sorted(R)})
    # join: follow the route keyed by the previous route's end state
    state, count = q0, 0
    for i, chunk in enumerate(chunks):
        if state == DEAD:
            break
        if not chunk:
            continue
        if state not in routes[i]:
            # C9: the arriving state has no transition on this chunk's first char
            assert delta(Tt, state, chunk[0]) == DEAD, "speculation unsound"
            state = DEAD
            break
        rt = routes[i][state]
        count += rt.hits
        state = rt.end
    accepted = state != DEAD and state in F
    return ParemRun(chunks, Rs, routes, state, accepted, count)


def compose(left: dict, right: dict) -> dict:
    """Associative join of two segment summaries {start: (end, hits)} keyed by start state
    (reading C5).  A missing right route means death (C9); DEAD is absorbing."""
    out = {}
    for q, (e, h) in left.items():
        if e == DEAD:
            out[q] = (DEAD, h)
        elif e in right:
            e2, h2 = right[e]
            out[q] = (e2, h + h2)
        else:
            out[q] = (DEAD, h)
    return out


def summary(Tt, F, chunk, starts) -> dict:
    F = set(F)
    return {r: (run_route(Tt, F, r, chunk).end, run_route(Tt, F, r, chunk).hits) for r in starts}
