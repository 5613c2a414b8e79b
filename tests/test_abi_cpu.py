"""CPU-only checks of the C ABI: the library loads, exports every symbol
include/jgs2.h declares, and the host-side symbolic analysis (nested
dissection front tree) is structurally valid. No device calls."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2506_06494_b200 import _lib as L
from paper_2506_06494_b200.model import box_grid

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "jgs2.h").read_text()
    return sorted(set(re.findall(r"\b(jgs2_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(L.EXPORTS)


def vertex_graph(tets, nv):
    pairs = set()
    for t in tets:
        for a in t:
            for b in t:
                pairs.add((int(a), int(b)))
    ptr = np.zeros(nv + 1, dtype=np.int64)
    adj = [[] for _ in range(nv)]
    for a, b in sorted(pairs):
        adj[a].append(b)
    for i in range(nv):
        ptr[i + 1] = ptr[i] + len(adj[i])
    return ptr, np.array([b for row in adj for b in row], dtype=np.int32)


def symbolic(ptr, adj, xyz, leaf):
    lib = L.lib()
    n = ptr.size - 1
    h = lib.jgs2_sym_build(n, L.ptr(ptr, L.i64), L.ptr(adj, L.i32), L.ptr(L.f64a(xyz), L.f64), leaf)
    assert h
    sizes = np.zeros(4, dtype=np.int64)
    L.check(lib.jgs2_sym_sizes(h, L.ptr(sizes, L.i64)))
    nf, ns = int(sizes[0]), int(sizes[1])
    out = dict(perm=np.zeros(n, np.int32), parent=np.zeros(nf, np.int32),
               cb=np.zeros(nf, np.int32), ce=np.zeros(nf, np.int32),
               sptr=np.zeros(nf + 1, np.int64), spos=np.zeros(max(ns, 1), np.int32),
               level=np.zeros(nf, np.int32))
    L.check(lib.jgs2_sym_export(h, *(L.ptr(out[k], L.i64 if k == "sptr" else L.i32)
                                     for k in ("perm", "parent", "cb", "ce", "sptr", "spos", "level"))))
    lib.jgs2_sym_free(h)
    out["nnz"] = int(sizes[3])
    return out


@pytest.mark.parametrize("div,leaf", [((6, 3, 2), 4), ((10, 6, 5), 16), ((3, 1, 1), 64)])
def test_nested_dissection_front_tree_covers_cholesky_pattern(div, leaf):
    mesh = box_grid(div, (1.0, 0.5, 0.4))
    nv = mesh.num_vertices
    ptr, adj = vertex_graph(mesh.tets, nv)
    S = symbolic(ptr, adj, mesh.rest_positions, leaf)
    perm = S["perm"]
    assert sorted(perm.tolist()) == list(range(nv))
    iperm = np.empty(nv, dtype=np.int64)
    iperm[perm] = np.arange(nv)
    nf = S["parent"].size
    owner = np.full(nv, -1)
    for f in range(nf):
        owner[S["cb"][f]:S["ce"][f]] = f
        assert S["parent"][f] == -1 or S["parent"][f] > f          # postorder
        if S["parent"][f] >= 0:
            assert S["level"][S["parent"][f]] > S["level"][f]
    assert np.all(owner >= 0)
    # symbolic Cholesky (vertex level) by elimination; every fill entry (i > j)
    # must lie in front(j)'s columns or its row structure.
    import scipy.sparse as sp
    A = sp.csr_matrix((np.ones(adj.size), adj, ptr), shape=(nv, nv))
    Ap = A[perm][:, perm].tolil()
    struct = [set() for _ in range(nv)]
    rows = [set(np.flatnonzero(Ap[:, j].toarray().ravel())) for j in range(nv)]
    for j in range(nv):
        s = {i for i in rows[j] if i > j} | struct[j]
        s.discard(j)
        if s:
            p = min(s)
            struct[p] |= {i for i in s if i > p}
        f = owner[j]
        allowed = set(range(S["cb"][f], S["ce"][f])) | set(S["spos"][S["sptr"][f]:S["sptr"][f + 1]].tolist())
        assert s <= allowed, (j, sorted(s - allowed)[:5])
