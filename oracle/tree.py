"""Medusa static trees (oracle; test infrastructure only).

A tree is given as a Medusa path list ("choices"): each element is the list of
top-k ranks from the root to a node, root implicit ("static, pre-built and
pruned attention trees"; SPEC.md path-list format).  Eq. 2 defines the
attention mask as the union of nodes on the S root-to-leaf paths; "prior to
verification, attention mask assumes full acceptance", i.e. node i sees
exactly its ancestors and itself.

Reading (R4/Q4): canonical node order = root, then sort by
(depth, lexicographic rank path).
"""
from __future__ import annotations

from dataclasses import dataclass, field


class InfeasibleTree(ValueError):
    pass


@dataclass
class Tree:
    paths: list[tuple[int, ...]]          # index n -> rank path of node n (root = ())
    topk: int
    parent: list[int] = field(default_factory=list)
    depth: list[int] = field(default_factory=list)
    rank: list[int] = field(default_factory=list)

    @property
    def N(self) -> int:
        return len(self.paths)

    @property
    def max_depth(self) -> int:
        return max(self.depth)

    def children(self, n: int) -> list[int]:
        return [c for c in range(self.N) if self.parent[c] == n]


def build(choices: list[list[int]], topk: int = 10) -> Tree:
    """Validate a path list and return the canonical tree.

    Errors (InfeasibleTree): duplicate path, orphan (a proper prefix missing),
    rank >= topk, negative rank, empty path.
    """
    seen = set()
    for p in choices:
        t = tuple(int(r) for r in p)
        if len(t) == 0:
            raise InfeasibleTree("empty path")
        if any(r < 0 or r >= topk for r in t):
            raise InfeasibleTree(f"rank out of range in {t}")
        if t in seen:
            raise InfeasibleTree(f"duplicate path {t}")
        seen.add(t)
    for t in seen:
        for j in range(1, len(t)):
            if t[:j] not in seen:
                raise InfeasibleTree(f"orphan path {t}: missing {t[:j]}")
    ordered = [()] + sorted(seen, key=lambda t: (len(t), t))
    index = {t: i for i, t in enumerate(ordered)}
    tree = Tree(paths=ordered, topk=topk)
    for t in ordered:
        tree.depth.append(len(t))
        tree.rank.append(t[-1] if t else -1)
        tree.parent.append(index[t[:-1]] if t else -1)
    return tree


def ancestors(tree: Tree, n: int) -> list[int]:
    """Ancestors of n from the root down (root first), excluding n."""
    out = []
    p = tree.parent[n]
    while p >= 0:
        out.append(p)
        p = tree.parent[p]
    return out[::-1]


def ancestor_mask(tree: Tree) -> list[list[int]]:
    """N x N 0/1 matrix, entry (i, j) = 1 iff j is i or an ancestor of i (Eq. 2)."""
    N = tree.N
    m = [[0] * N for _ in range(N)]
    for i in range(N):
        m[i][i] = 1
        for j in ancestors(tree, i):
            m[i][j] = 1
    return m


def leaves(tree: Tree) -> list[int]:
    """Leaf node ids in DFS (lexicographic rank-path) order."""
    has_child = [False] * tree.N
    for c in range(1, tree.N):
        has_child[tree.parent[c]] = True
    ls = [n for n in range(tree.N) if not has_child[n]]
    return sorted(ls, key=lambda n: tree.paths[n])


def dfs_order(tree: Tree) -> list[int]:
    """All node ids in DFS pre-order (lexicographic rank path)."""
    return sorted(range(tree.N), key=lambda n: tree.paths[n])


def candidate_paths(tree: Tree) -> list[list[int]]:
    """S candidate sequences as node-id lists root..leaf, padded with -1 to
    length max_depth+1 ("total candidate sequences S")."""
    L = tree.max_depth + 1
    out = []
    for leaf in leaves(tree):
        ids = ancestors(tree, leaf) + [leaf]
        out.append(ids + [-1] * (L - len(ids)))
    return out


def level_counts(tree: Tree) -> list[int]:
    cnt = [0] * (tree.max_depth + 1)
    for d in tree.depth:
        cnt[d] += 1
    return cnt


def stats(tree: Tree) -> dict:
    """(N, S, l) and the per-level label, e.g. '1-10-23-23-7'."""
    return dict(N=tree.N, S=len(leaves(tree)), depth=tree.max_depth,
                label="-".join(str(c) for c in level_counts(tree)))


def truncate(choices: list[list[int]], depth: int) -> list[list[int]]:
    """Keep nodes of depth <= ``depth`` (a Medusa tree used with fewer heads)."""
    return [list(p) for p in choices if len(p) <= depth]


def prune_right_to_left(choices: list[list[int]], target_nodes: int, topk: int = 10) -> list[list[int]]:
    """Reading R4 of P:247 ("Medusa's right-to-left pruning"): repeatedly delete
    the leaf whose rank path is lexicographically largest (the rightmost leaf in
    DFS order) until ``target_nodes`` nodes (root included) remain."""
    tree = build(choices, topk)
    if target_nodes < 1 or target_nodes > tree.N:
        raise InfeasibleTree("target outside [1, N]")
    cur = set(tuple(p) for p in choices)
    while len(cur) + 1 > target_nodes:
        lv = [t for t in cur if not any(len(u) == len(t) + 1 and u[:len(t)] == t for u in cur)]
        cur.remove(max(lv))
    return [list(t) for t in sorted(cur, key=lambda t: (len(t), t))]


# ----------------------------------------------------------------- f1: SpecMemo tree construction
def full_tree(k: int, l: int) -> list[list[int]]:
    """Full k-ary tree of depth l as a path list: Eq. 2's N = sum_{i=0}^{l} k^i nodes."""
    out, level = [], [[]]
    for _ in range(l):
        level = [p + [r] for p in level for r in range(k)]
        out += level
    return out


def prune_rate(level: int, r_min: float = 0.1, r_max: float = 0.95, mid: float = 2.5, steep: float = 2.0) -> float:
    """Scaled logistic per-level pruning rate (fig:prunefunc; "low at first levels
    ... increase the rate on deeper levels"):  r(i) = r_min + (r_max - r_min) / (1 + exp(-steep (i - mid))).
    The four parameters are unreadable in the paper (an image): parity unpinned; defaults = SPEC S:220."""
    import math
    return r_min + (r_max - r_min) / (1.0 + math.exp(-steep * (level - mid)))


def prune_full_tree(k: int, l: int, r_min=0.1, r_max=0.95, mid=2.5, steep=2.0) -> list[list[int]]:
    """Custom tree build via pruning: level 1 keeps all k nodes (first-level rule);
    level i >= 2 keeps the first ceil((1 - r(i)) * k^i) nodes of the full tree's level, left to right
    (lexicographic rank path = highest-probability tokens first), minus those whose parent was dropped."""
    import math
    kept = [[r] for r in range(k)] if l >= 1 else []
    prev = set(tuple(p) for p in kept)
    for i in range(2, l + 1):
        n_i = math.ceil((1.0 - prune_rate(i, r_min, r_max, mid, steep)) * k ** i - 1e-9)
        level = [list(p) + [r] for p in sorted(prev) for r in range(k)]  # left to right
        level = level[:n_i]
        kept += level
        prev = set(tuple(p) for p in level)
        if not prev:
            break
    return kept


def build_custom_tree(n_nodes: int, n_leaves: int, k: int, l: int) -> list[list[int]]:
    """Custom tree build from tree features (Alg. 1's (N, S) pairs) -- the
    construction rule is not in the paper (reading Q30): start from the root and
    c1 = min(k, N-1, S) level-1 nodes; then add the remaining nodes one at a time:
      (a) N - 1 - c1 - (S - c1) "deepening" additions first: a child of the first leaf in DFS
          order whose depth < l (leaf count unchanged), so depth concentrates on the left;
      (b) then "widening" additions: the next-rank child of the first node in BFS order (shallowest,
          then leftmost) that already has children and fewer than k (one more leaf each); a
          widening step is taken early only when every leaf already sits at depth l.
    Raises InfeasibleTree when (N, S, k, l) admits no tree under this rule."""
    N, S = n_nodes, n_leaves
    if N < 1 or S < 1 or (N == 1 and S != 1) or S > N - 1 + (N == 1):
        raise InfeasibleTree("need 1 <= S <= N - 1 (or N = S = 1)")
    if N == 1:
        return []
    c1 = min(k, N - 1, S)
    paths = [[r] for r in range(c1)]
    children = {(): c1}
    leaves_now = c1
    widen = S - leaves_now
    deepen = (N - 1 - c1) - widen
    if widen < 0 or deepen < 0:
        raise InfeasibleTree("(N, S) not reachable: too many leaves for the nodes")

    def sorted_paths():
        return sorted(paths)                                            # DFS = lexicographic

    def widen_one():
        internal = sorted((p for p in [[]] + paths if 0 < children.get(tuple(p), 0) < k), key=lambda p: (len(p), p))
        if not internal:
            raise InfeasibleTree("no internal node with free arity to widen")
        p = internal[0]
        r = children[tuple(p)]
        paths.append(p + [r])
        children[tuple(p)] = r + 1

    while deepen > 0:
        cands = [p for p in sorted_paths() if len(p) < l and children.get(tuple(p), 0) == 0]
        if cands:                      # deepening preferred
            p = cands[0]
            paths.append(p + [0])
            children[tuple(p)] = 1
            deepen -= 1
        elif widen > 0:                # every leaf is at depth l: widen once, then deepen again
            widen_one()
            widen -= 1
        else:
            raise InfeasibleTree("no leaf above depth l to deepen")
    for _ in range(widen):
        widen_one()
    return sorted(paths, key=lambda p: (len(p), p))


# ----------------------------------------------------------------- tree-size selection (f1)
def expected_tau(choices: list[list[int]], alpha, rho: float = 1.0, topk: int = 10) -> float:
    """Expected acceptance length tau of a tree under the independent acceptance model of
    SPEC's simulator (AcceptanceModel): the non-root node at level j with sibling
    rank r is accepted with probability alpha_j * rho^r, independently; the accepted path is the
    longest root path whose nodes are all accepted ("the longest candidate sequence that
    verified its tokens is accepted"); tau = its depth + 1 (reading Q12).

    E[tau] = 1 + sum_{D=1}^{l} P(max accepted depth >= D), and P(max >= D) = f_D(root) with
    f_D(n) = 1 if depth(n) >= D, else 1 - prod_{c child of n} (1 - a(c) f_D(c))
    (a path reaching depth D exists below n iff some child is accepted and has one below it)."""
    t = build(choices, topk)
    a = [0.0] + [float(alpha[t.depth[n] - 1]) * float(rho) ** t.rank[n] for n in range(1, t.N)]
    kids = [[] for _ in range(t.N)]
    for n in range(1, t.N):
        kids[t.parent[n]].append(n)
    tau = 1.0
    for D in range(1, t.max_depth + 1):
        f = [0.0] * t.N
        for n in reversed(range(t.N)):          # canonical order lists parents before children
            if t.depth[n] >= D:
                f[n] = 1.0
            else:
                miss = 1.0
                for c in kids[n]:
                    miss *= 1.0 - a[c] * f[c]
                f[n] = 1.0 - miss
        tau += f[0]
    return tau


def select_tree(candidates: list[list[list[int]]], step_ms, alpha, rho: float = 1.0, batch: int = 1,
                topk: int = 10) -> tuple[int, list[float]]:
    """Tree-size selection (the paper's choice of heads x mask by measured
    per-token latency, fig:maskmodel P:326-401, "3 heads with mask of size 44 gives the best
    latency" P:399): expected decode throughput of candidate i = batch * E[tau_i] / step_ms[i]
    (tokens per ms); pick the largest, ties to fewer nodes, then the lower index.
    Returns (index, per-candidate expected tokens/s)."""
    tps = [batch * expected_tau(c, alpha, rho, topk) / float(step_ms[i]) * 1e3 for i, c in enumerate(candidates)]
    best = 0
    for i in range(1, len(candidates)):
        if tps[i] > tps[best] or (tps[i] == tps[best] and len(candidates[i]) < len(candidates[best])):
            best = i
    return best, tps
