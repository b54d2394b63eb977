"""Sequential trace oracle of the expert registry (TEST INFRASTRUCTURE ONLY).

Restates SPEC.md:463-514 (registry module; the reference ships no registry code):
strict LRU over unpinned residents with logical ticks, pin counts, whole-artifact loads,
"budget exceeded" leaves the state unchanged.  `replay(ops)` returns the observable
outcome of every operation so the product registry can be checked against it.
"""

from __future__ import annotations


class OracleRegistry:
    def __init__(self, budget: int):
        self.budget = budget
        self.size = {}       # id -> bytes (registered)
        self.resident = {}   # id -> [last_use_tick, pins]
        self.tick = 0
        self.current = 0
        self.peak = 0
        self.loads = 0
        self.evicts = 0

    def register(self, eid, size):
        if eid in self.size:
            return ("error", "duplicate")
        if size > self.budget:
            return ("error", "budget")
        self.size[eid] = size
        return ("ok",)

    def acquire(self, eid):
        """returns ('hit',) | ('load', victims) | ('error', kind)."""
        if eid not in self.size:
            return ("error", "unknown")
        self.tick += 1
        if eid in self.resident:
            r = self.resident[eid]
            r[0] = self.tick
            r[1] += 1
            return ("hit",)
        need = self.size[eid]
        victims = []
        free = self.budget - self.current
        cands = sorted((r[0], k) for k, r in self.resident.items() if r[1] == 0)
        for _, k in cands:
            if free >= need:
                break
            victims.append(k)
            free += self.size[k]
        if free < need:
            self.tick -= 1
            return ("error", "budget")
        for k in victims:
            del self.resident[k]
            self.current -= self.size[k]
            self.evicts += 1
        self.resident[eid] = [self.tick, 1]
        self.current += need
        self.loads += 1
        self.peak = max(self.peak, self.current)
        return ("load", tuple(victims))

    def release(self, eid):
        r = self.resident.get(eid)
        if r is None or r[1] == 0:
            return ("error", "not acquired")
        r[1] -= 1
        return ("ok",)


def replay(budget, ops):
    """ops: ('register', id, size) | ('acquire', id) | ('release', id) -> list of outcomes."""
    o = OracleRegistry(budget)
    out = []
    for op in ops:
        if op[0] == "register":
            out.append(o.register(op[1], op[2]))
        elif op[0] == "acquire":
            out.append(o.acquire(op[1]))
        else:
            out.append(o.release(op[1]))
    return out, o
