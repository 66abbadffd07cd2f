"""Offline study of elimination orders on a coupling graph dumped by the Cholesky
analysis (ABD_CHOL_DUMP_GRAPH=file): fill, update pairs, elimination-tree height and
a critical-path estimate for the orders the analysis could use.

    python tools/chol_order_study.py GRAPH.bin
"""
import heapq
import sys

import numpy as np


def load(path):
    raw = open(path, "rb").read()
    n = int(np.frombuffer(raw, np.int32, 1, 0)[0])
    ne = int(np.frombuffer(raw, np.int64, 1, 4)[0])
    e = np.frombuffer(raw, np.uint64, ne, 12)
    return n, np.stack([(e >> np.uint64(32)).astype(np.int64), (e & np.uint64(0xffffffff)).astype(np.int64)], 1)


def local_graph(edges):
    nodes = np.unique(edges.ravel())
    loc = {int(g): i for i, g in enumerate(nodes)}
    adj = [set() for _ in nodes]
    for a, b in edges:
        adj[loc[int(a)]].add(loc[int(b)])
        adj[loc[int(b)]].add(loc[int(a)])
    return nodes, adj


def contract(adj):
    """rake / compress rounds as chol_analyze (k_chol.cu); returns (order, remaining core adj dict)"""
    m = len(adj)
    a = [set(s) for s in adj]
    gone = [False] * m
    live = list(range(m))
    order = []
    while True:
        prog = False
        sel = [v for v in live if len(a[v]) <= 1]
        for v in sel:
            if gone[v]:
                continue
            for u in a[v]:
                a[u].discard(v)
            a[v] = set()
            gone[v] = True
            order.append(v)
            prog = True
        blocked = set()
        sel = []
        for v in live:
            if not gone[v] and v not in blocked and len(a[v]) == 2:
                x, y = sorted(a[v])
                sel.append(v)
                blocked |= {v, x, y}
        for v in sel:
            x, y = list(a[v])
            a[x].discard(v)
            a[y].discard(v)
            a[x].add(y)
            a[y].add(x)
            a[v] = set()
            gone[v] = True
            order.append(v)
            prog = True
        live = [v for v in live if not gone[v]]
        if not prog or not live:
            break
    return order, {v: set(a[v]) for v in live}


def min_degree(core, nodes=None):
    a = {v: set(s) for v, s in core.items()} if nodes is None else {v: core[v] & nodes for v in nodes}
    heap = [(len(s), v) for v, s in a.items()]
    heapq.heapify(heap)
    done, order = set(), []
    while heap:
        d, v = heapq.heappop(heap)
        if v in done or d != len(a[v]):
            continue
        done.add(v)
        order.append(v)
        nb = a[v]
        for u in nb:
            a[u] |= nb
            a[u].discard(u)
            a[u].discard(v)
            heapq.heappush(heap, (len(a[u]), u))
    return order


def bisect(a, nodes):
    """BFS level-structure separator from a pseudo-peripheral node: the middle level"""
    nodes = set(nodes)
    start = min(nodes)
    for _ in range(3):
        lv = {start: 0}
        fr = [start]
        while fr:
            nf = []
            for v in fr:
                for u in a[v]:
                    if u in nodes and u not in lv:
                        lv[u] = lv[v] + 1
                        nf.append(u)
            if nf:
                last = nf
            fr = nf
        if len(lv) < len(nodes):  # disconnected: split off this component
            comp = set(lv)
            return comp, nodes - comp, set()
        start = min(last)
    dmax = max(lv.values())
    if dmax < 2:
        return None
    # choose the level that best balances the two sides
    cnt = np.bincount(list(lv.values()))
    cum = np.cumsum(cnt)
    best, bl = None, None
    for L in range(1, dmax):
        left, right = cum[L - 1], len(nodes) - cum[L]
        score = max(left, right) + 2 * cnt[L]
        if best is None or score < best:
            best, bl = score, L
    sep = {v for v, l in lv.items() if l == bl}
    A = {v for v, l in lv.items() if l < bl}
    B = {v for v, l in lv.items() if l > bl}
    return A, B, sep


def nested_dissection(core, leaf=32):
    order = []

    def rec(nodes):
        if len(nodes) <= leaf:
            order.extend(min_degree(core, set(nodes)))
            return
        r = bisect(core, nodes)
        if r is None:
            order.extend(min_degree(core, set(nodes)))
            return
        A, B, S = r
        if A:
            rec(A)
        if B:
            rec(B)
        order.extend(sorted(S))

    rec(set(core))
    return order


def symbolic(adj, order):
    m = len(adj)
    pos = np.empty(m, np.int64)
    pos[order] = np.arange(m)
    cs = [None] * m
    children = [[] for _ in range(m)]
    for v in order:
        s = {u for u in adj[v] if pos[u] > pos[v]}
        for c in children[v]:
            s |= set(cs[c])
        s.discard(v)
        cs[v] = sorted(s, key=lambda u: pos[u])
        if cs[v]:
            children[cs[v][0]].append(v)
    return pos, cs


def evaluate(name, adj, order, t_node=11.0, t_prod=0.15):
    pos, cs = symbolic(adj, order)
    m = len(adj)
    nnz = sum(len(c) for c in cs)
    upd = sum(len(c) * (len(c) - 1) // 2 for c in cs)
    rows = np.zeros(m, np.int64)
    for v in range(m):
        for u in cs[v]:
            rows[u] += 1
    h = np.zeros(m, np.int64)
    cp = np.zeros(m)
    for v in order:
        # node latency: fixed chain (diag + block) + its heaviest serial product chain
        upd_max = 0
        for i, u in enumerate(cs[v]):
            upd_max = max(upd_max, 0)
        c = t_node + t_prod * rows[v]
        cp[v] += c
        if cs[v]:
            p = cs[v][0]
            h[p] = max(h[p], h[v] + 1)
            cp[p] = max(cp[p], cp[v])
    print(f"{name:24s} m={m} L_off={nnz} upd={upd} height={h.max() + 1} critpath~{cp.max():.0f} us "
          f"maxrow={rows.max()} maxcol={max(len(c) for c in cs)}")
    return h, cs


def main():
    n, edges = load(sys.argv[1])
    nodes, adj = local_graph(edges)
    print(f"n={n} coupled={len(nodes)} edges={len(edges)}")
    corder, core = contract(adj)
    print(f"contracted {len(corder)}, core {len(core)}")
    evaluate("rake/compress + MD", adj, corder + min_degree(core))
    for leaf in (8, 16, 32, 64):
        evaluate(f"rake/compress + ND{leaf}", adj, corder + nested_dissection(core, leaf))
    evaluate("MD (whole graph)", adj, min_degree({v: s for v, s in enumerate(adj)}))


if __name__ == "__main__":
    main()
