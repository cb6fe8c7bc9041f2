"""Dump the K2 unit graph (pieces: boundary vertices of one connected part of
a component, see bg_order.hpp) of a BASELINE config for tools/k2_layout_sim:
  u32 nu | u64 bsize[nu] | u64 nadj | (u32, u32) adj[nadj]
Usage: python tools/k2_units.py delaunay262k_k256 /tmp/units.bin"""
import sys, os
import numpy as np
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import graphs

g, cfg = graphs.make(sys.argv[1])
a = P.partition_graph(g, cfg["k"], 0, os.cpu_count() or 8).astype(np.int64)
eu, ev = g.eu.astype(np.int64), g.ev.astype(np.int64)
cross = a[eu] != a[ev]
bnd = np.zeros(g.n, bool)
bnd[eu[cross]] = True
bnd[ev[cross]] = True
intra = ~cross
ncc, lab = connected_components(coo_matrix((np.ones(intra.sum()), (eu[intra], ev[intra])), shape=(g.n, g.n)),
                                directed=False)
# units: connected parts holding boundary vertices, numbered in order of first boundary vertex
ub = lab[bnd]
uniq, unit_of_b = np.unique(ub, return_inverse=True)
nu = len(uniq)
bsize = np.bincount(unit_of_b, minlength=nu).astype(np.uint64)
uid = -np.ones(ncc, np.int64)
uid[uniq] = np.arange(nu)
pu, pv = uid[lab[eu[cross]]], uid[lab[ev[cross]]]
pairs = np.unique(np.stack([pu, pv], 1), axis=0)
with open(sys.argv[2], "wb") as f:
    np.array([nu], np.uint32).tofile(f)
    bsize.tofile(f)
    np.array([len(pairs)], np.uint64).tofile(f)
    pairs.astype(np.uint32).tofile(f)
print(f"{sys.argv[1]}: b={int(bsize.sum())} units={nu} unit edges={len(pairs)}")
