"""And-Inverter Graph with one-level structural hashing and constant folding.

The paper optimises its FloPoCo netlists with ABC's ``strash`` (AIG by
one-level structural hashing) before mapping them onto the target's bitwise
cells.  This is the in-repo equivalent: every circuit the
generator builds is created directly as a structurally hashed AIG.

Literals: ``lit = 2 * node + complement``; node 0 is constant false, so
``FALSE = 0`` and ``TRUE = 1``.  Node ids are created in topological order.
"""
from __future__ import annotations

FALSE = 0
TRUE = 1


def lit_not(a: int) -> int:
    return a ^ 1


class AIG:
    def __init__(self):
        self.f0 = [0]          # fanin literal 0 of each node (0 for const / input)
        self.f1 = [0]
        self.kind = ["const"]  # "const" | "input" | "and"
        self.input_names: list[str] = []
        self.input_nodes: list[int] = []
        self._hash: dict[tuple[int, int], int] = {}

    # ----------------------------------------------------------------- nodes
    def n_nodes(self) -> int:
        return len(self.f0)

    def input(self, name: str) -> int:
        node = len(self.f0)
        self.f0.append(0)
        self.f1.append(0)
        self.kind.append("input")
        self.input_names.append(name)
        self.input_nodes.append(node)
        return 2 * node

    def inputs(self, name: str, n: int) -> list[int]:
        return [self.input(f"{name}[{i}]") for i in range(n)]

    def AND(self, a: int, b: int) -> int:
        # constant folding and trivial identities
        if a == FALSE or b == FALSE or a == (b ^ 1):
            return FALSE
        if a == TRUE:
            return b
        if b == TRUE or a == b:
            return a
        if a > b:
            a, b = b, a
        # two-level simplifications: a & (a & x) = a & x ; a & (~a & x) = 0
        for x, y in ((a, b), (b, a)):
            ny = y >> 1
            if not (y & 1) and self.kind[ny] == "and":
                p, q = self.f0[ny], self.f1[ny]
                if x == p or x == q:
                    return y
                if x == (p ^ 1) or x == (q ^ 1):
                    return FALSE
        key = (a, b)
        node = self._hash.get(key)
        if node is None:
            node = len(self.f0)
            self.f0.append(a)
            self.f1.append(b)
            self.kind.append("and")
            self._hash[key] = node
        return 2 * node

    # ----------------------------------------------------------------- derived gates
    def NOT(self, a: int) -> int:
        return a ^ 1

    def OR(self, a: int, b: int) -> int:
        return self.AND(a ^ 1, b ^ 1) ^ 1

    def XOR(self, a: int, b: int) -> int:
        if a == FALSE:
            return b
        if b == FALSE:
            return a
        if a == TRUE:
            return b ^ 1
        if b == TRUE:
            return a ^ 1
        if a == b:
            return FALSE
        if a == (b ^ 1):
            return TRUE
        return self.OR(self.AND(a, b ^ 1), self.AND(a ^ 1, b))

    def XNOR(self, a: int, b: int) -> int:
        return self.XOR(a, b) ^ 1

    def MUX(self, s: int, a: int, b: int) -> int:
        """s ? a : b"""
        if s == TRUE:
            return a
        if s == FALSE:
            return b
        if a == b:
            return a
        if a == TRUE and b == FALSE:
            return s
        if a == FALSE and b == TRUE:
            return s ^ 1
        return self.OR(self.AND(s, a), self.AND(s ^ 1, b))

    def MAJ(self, a: int, b: int, c: int) -> int:
        for x, y, z in ((a, b, c), (b, c, a), (c, a, b)):
            if x == FALSE:
                return self.AND(y, z)
            if x == TRUE:
                return self.OR(y, z)
        return self.OR(self.AND(a, b), self.AND(c, self.OR(a, b)))

    def XOR3(self, a: int, b: int, c: int) -> int:
        return self.XOR(self.XOR(a, b), c)

    def OR_many(self, xs) -> int:
        xs = [x for x in xs if x != FALSE]
        if any(x == TRUE for x in xs):
            return TRUE
        if not xs:
            return FALSE
        while len(xs) > 1:
            nxt = []
            for i in range(0, len(xs) - 1, 2):
                nxt.append(self.OR(xs[i], xs[i + 1]))
            if len(xs) % 2:
                nxt.append(xs[-1])
            xs = nxt
        return xs[0]

    def AND_many(self, xs) -> int:
        return self.OR_many([x ^ 1 for x in xs]) ^ 1

    # ----------------------------------------------------------------- evaluation
    def simulate(self, input_words: dict, outputs: list[int], np):
        """Word-parallel simulation (numpy uint64 arrays): returns list of output words."""
        vals = [None] * self.n_nodes()
        shape = next(iter(input_words.values())).shape
        zero = np.zeros(shape, dtype=np.uint64)
        vals[0] = zero
        for name, node in zip(self.input_names, self.input_nodes):
            vals[node] = input_words[name]
        ones = ~zero

        def lv(l):
            v = vals[l >> 1]
            return (v ^ ones) if (l & 1) else v

        for n in range(1, self.n_nodes()):
            if self.kind[n] == "and":
                vals[n] = lv(self.f0[n]) & lv(self.f1[n])
        return [lv(o) for o in outputs]
