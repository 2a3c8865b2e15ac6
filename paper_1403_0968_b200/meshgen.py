"""Seeded synthetic input generator (meshes and fields), shared by the tests,
the oracle leg and the CUDA leg.

It holds none of the method's arithmetic: no GLL nodes, no differentiation, no
geometric factors, no assembly.  The 1-D reference node positions ``r1d`` are
an *argument* (tests pass the oracle's GLL nodes, the product path passes the
library's), so the same recipe feeds both sides without either importing the
other.

Recipe: a Nekbone-shaped brick box of
ex x ey x ez conforming hexahedra on [0,Lx]x[0,Ly]x[0,Lz]; GLL nodes mapped
affinely into each element and then deformed by
    x <- x + eps * min(L) * S(x) * (1, 0.5, -0.7),
    S = sin(pi x/Lx) sin(pi y/Ly) sin(pi z/Lz)     (pre-deformation coordinates)
so shared nodes get bit-identical coordinates in every element that holds
them and the boundary stays planar.  Global ids follow the lexicographic
global node grid (Fischer-style global-local numbering);
homogeneous Dirichlet on every box face (reading G7).

Local storage is element-major, node (i,j,k) at e*n^3 + i + n*j + n*n*k.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Mesh:
    N: int
    xyz: np.ndarray         # [E, 3, n^3] float64
    glo: np.ndarray         # [E, n^3] int64 global node ids (consistent across ranks)
    dirichlet: np.ndarray   # [E, n^3] uint8, 1 = Dirichlet node
    elems: tuple            # global element grid (ex, ey, ez)
    lengths: tuple          # box lengths
    parts: tuple = (1, 1, 1)
    rank: int = 0
    eidx: np.ndarray = field(default=None)   # [E, 3] global element (a, b, c)
    nboundary: int = 0      # leading elements that touch a partition interface

    @property
    def nelem(self) -> int:
        return int(self.glo.shape[0])

    @property
    def nlocal(self) -> int:
        return int(self.glo.size)

    @property
    def nglobal(self) -> int:
        """Number of distinct global ids (for a box: (ex N + 1)(ey N + 1)(ez N + 1))."""
        return int(np.unique(self.glo).size)


def rank_block(elems, parts, rank):
    """Element index ranges [lo, hi) per axis owned by ``rank`` (x fastest)."""
    px, py, pz = parts
    rx = rank % px
    ry = (rank // px) % py
    rz = rank // (px * py)
    out = []
    for e, p, r in zip(elems, (px, py, pz), (rx, ry, rz)):
        lo = (e * r) // p
        hi = (e * (r + 1)) // p
        out.append((lo, hi))
    return out


def default_parts(nranks: int):
    """3-D block partition minimising surface."""
    table = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}
    if nranks in table:
        return table[nranks]
    return (1, 1, nranks)


def box_mesh(N: int, r1d, elems=(2, 2, 2), lengths=(1.0, 1.0, 1.0), eps: float = 0.0,
             parts=(1, 1, 1), rank: int = 0, boundary_first: bool = False,
             dirichlet_faces: bool = True) -> Mesh:
    """dirichlet_faces=False: no Dirichlet nodes (natural boundary; the
    screened operator with alpha > 0 is SPD without a mask)."""
    r1d = np.asarray(r1d, dtype=np.float64)
    n = N + 1
    assert r1d.shape == (n,), "r1d must hold the N+1 reference node positions"
    ex, ey, ez = elems
    Lx, Ly, Lz = (float(v) for v in lengths)
    (ax0, ax1), (by0, by1), (cz0, cz1) = rank_block(elems, parts, rank)
    a, b, c = np.meshgrid(np.arange(ax0, ax1), np.arange(by0, by1), np.arange(cz0, cz1),
                          indexing="ij")
    # element order: a fastest, then b, then c
    a = a.transpose(2, 1, 0).reshape(-1)
    b = b.transpose(2, 1, 0).reshape(-1)
    c = c.transpose(2, 1, 0).reshape(-1)
    eidx = np.stack([a, b, c], axis=1)
    nb = 0
    if boundary_first and tuple(parts) != (1, 1, 1):
        touch = np.zeros(len(a), dtype=bool)
        for v, lo, hi, e in ((a, ax0, ax1, ex), (b, by0, by1, ey), (c, cz0, cz1, ez)):
            touch |= (v == lo) & (lo > 0)
            touch |= (v == hi - 1) & (hi < e)
        order = np.concatenate([np.nonzero(touch)[0], np.nonzero(~touch)[0]])
        nb = int(touch.sum())
        eidx = eidx[order]
        a, b, c = eidx[:, 0], eidx[:, 1], eidx[:, 2]
    # local node (i,j,k), i fastest
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i = i.reshape(-1)
    j = j.reshape(-1)
    k = k.reshape(-1)
    I = a[:, None] * N + i[None, :]
    J = b[:, None] * N + j[None, :]
    K = c[:, None] * N + k[None, :]
    nx, ny = ex * N + 1, ey * N + 1
    glo = (I + nx * (J + ny * K)).astype(np.int64)
    dirichlet = ((I == 0) | (I == ex * N) | (J == 0) | (J == ey * N) |
                 (K == 0) | (K == ez * N)).astype(np.uint8)
    if not dirichlet_faces:
        dirichlet[:] = 0
    # affine placement: x = (a + (1 + r_i)/2) * hx  (exact at shared faces)
    x = (a[:, None] + (1.0 + r1d[i])[None, :] / 2.0) * (Lx / ex)
    y = (b[:, None] + (1.0 + r1d[j])[None, :] / 2.0) * (Ly / ey)
    z = (c[:, None] + (1.0 + r1d[k])[None, :] / 2.0) * (Lz / ez)
    if eps != 0.0:
        S = np.sin(np.pi * x / Lx) * np.sin(np.pi * y / Ly) * np.sin(np.pi * z / Lz)
        amp = eps * min(Lx, Ly, Lz)
        x, y, z = x + amp * S, y + 0.5 * amp * S, z - 0.7 * amp * S
    xyz = np.stack([x, y, z], axis=1)
    return Mesh(N=N, xyz=np.ascontiguousarray(xyz), glo=np.ascontiguousarray(glo),
                dirichlet=np.ascontiguousarray(dirichlet), elems=tuple(elems),
                lengths=(Lx, Ly, Lz), parts=tuple(parts), rank=rank, eidx=eidx,
                nboundary=nb)


def random_field(n: int, seed: int) -> np.ndarray:
    """u ~ U(-1, 1), numpy default_rng(seed)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def manufactured(mesh: Mesh):
    """u* = prod sin(pi x_c / L_c) (vanishes on the box faces) and
    f = -Laplace u* = pi^2 (1/Lx^2 + 1/Ly^2 + 1/Lz^2) u*, at the nodes."""
    Lx, Ly, Lz = mesh.lengths
    x, y, z = mesh.xyz[:, 0], mesh.xyz[:, 1], mesh.xyz[:, 2]
    us = np.sin(np.pi * x / Lx) * np.sin(np.pi * y / Ly) * np.sin(np.pi * z / Lz)
    f = math.pi ** 2 * (1 / Lx ** 2 + 1 / Ly ** 2 + 1 / Lz ** 2) * us
    return us.reshape(-1), f.reshape(-1)


def cube_poly(mesh: Mesh):
    """u* = x(1-x) y(1-y) z(1-z) on the unit cube (degree 2 per direction) and
    f = -Laplace u* = 2[y(1-y)z(1-z) + x(1-x)z(1-z) + x(1-x)y(1-y)]."""
    x, y, z = mesh.xyz[:, 0], mesh.xyz[:, 1], mesh.xyz[:, 2]
    gx, gy, gz = x * (1 - x), y * (1 - y), z * (1 - z)
    us = gx * gy * gz
    f = 2.0 * (gy * gz + gx * gz + gx * gy)
    return us.reshape(-1), f.reshape(-1)


def coefficients(mesh: Mesh, kappa_amp: float = 0.5, alpha0: float = 1.0):
    """Smooth material coefficients of the screened-Coulomb workload (NEXT-1,
    eq:semPDE kappa(x), alpha(x)), evaluated at the node coordinates (so every
    copy of a shared node gets the same values):
        kappa = 1 + a sin(2 pi x/Lx) cos(pi y/Ly) cos(2 pi z/Lz)   in [1-a, 1+a]
        alpha = alpha0 (1 + 0.5 cos(pi x/Lx) cos(pi y/Ly))          in [alpha0/2, 3 alpha0/2]
    Returns (kappa, alpha), each [E * n^3]."""
    Lx, Ly, Lz = mesh.lengths
    x, y, z = mesh.xyz[:, 0], mesh.xyz[:, 1], mesh.xyz[:, 2]
    kappa = 1.0 + kappa_amp * (np.sin(2 * np.pi * x / Lx) * np.cos(np.pi * y / Ly)
                               * np.cos(2 * np.pi * z / Lz))
    alpha = alpha0 * (1.0 + 0.5 * np.cos(np.pi * x / Lx) * np.cos(np.pi * y / Ly))
    return np.ascontiguousarray(kappa.reshape(-1)), np.ascontiguousarray(alpha.reshape(-1))


def relabel(mesh: Mesh, seed: int, rotate: bool = True, id_stride: int = 3) -> Mesh:
    """The same discretisation presented differently (robustness inputs; no
    method arithmetic): elements in a random order, each element's local
    nodes turned by a random quarter rotation about its k axis,
    (i, j, k) <- (N - j, i, k) applied 0-3 times (orientation preserving, so
    J stays > 0), and the global ids replaced by a random injective relabelling
    with gaps (id -> id_stride * perm(id) + 7, a non-compact id range).
    Returns a new Mesh (nboundary = 0)."""
    rng = np.random.default_rng(seed)
    n = mesh.N + 1
    n3 = n ** 3
    E = mesh.nelem
    order = rng.permutation(E)
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.reshape(-1), j.reshape(-1), k.reshape(-1)
    rots = [np.arange(n3)]
    ii, jj = i.copy(), j.copy()
    for _ in range(3):
        ii, jj = mesh.N - jj, ii                  # new node (i,j,k) takes old (N-j, i, k)
        rots.append(ii + n * jj + n * n * k)
    which = rng.integers(0, 4 if rotate else 1, size=E)
    xyz = np.empty_like(mesh.xyz)
    glo = np.empty_like(mesh.glo)
    dirichlet = np.empty_like(mesh.dirichlet)
    for new_e, old_e in enumerate(order):
        src = rots[which[new_e]]
        xyz[new_e] = mesh.xyz[old_e][:, src]
        glo[new_e] = mesh.glo[old_e][src]
        dirichlet[new_e] = mesh.dirichlet[old_e][src]
    ids = np.unique(mesh.glo)
    perm = rng.permutation(ids.size)
    remap = np.empty(int(ids.max()) + 1, dtype=np.int64)
    remap[ids] = id_stride * perm.astype(np.int64) + 7
    glo = remap[glo]
    eidx = None if mesh.eidx is None else mesh.eidx[order]
    return Mesh(N=mesh.N, xyz=np.ascontiguousarray(xyz), glo=np.ascontiguousarray(glo),
                dirichlet=np.ascontiguousarray(dirichlet), elems=mesh.elems, lengths=mesh.lengths,
                parts=mesh.parts, rank=mesh.rank, eidx=eidx, nboundary=0)


def prism_mesh(N: int, r1d, sides: int = 3, nz: int = 2, height: float = 1.0,
               radius: float = 1.0) -> Mesh:
    """A NON-box conforming hexahedral mesh (Omega_h is any
    union of E conforming hexahedra): a regular `sides`-gon of the given
    radius split into `sides` quadrilaterals around its centre -- quad q has
    the corners (centre, midpoint of edge (q-1, q), vertex q, midpoint of edge
    (q, q+1)), counter-clockwise -- extruded over `nz` layers in z.  The
    vertical edge through the centre is shared by `sides` hexahedra, so edge
    nodes there have multiplicity sides (3, 5, 6, ...) and the interior
    corner nodes on it 2*sides -- multiplicities a box never has.  GLL nodes
    are placed by the bilinear map of each quad (elements are kites, not
    parallelograms: all six geometric factors vary in the element) and
    linearly in z.  Global ids: nodes with the same coordinates (to 1e-9 of
    the radius) are one node; the coordinates of each global node are taken
    from its first copy so every copy is bit-identical.  Dirichlet on every
    boundary face (faces not shared by two elements).  Element order: layer by
    layer, quads in angular order."""
    r1d = np.asarray(r1d, dtype=np.float64)
    n = N + 1
    assert r1d.shape == (n,)
    ang = 2.0 * np.pi * np.arange(sides) / sides
    V = radius * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    Mid = 0.5 * (V + np.roll(V, -1, axis=0))          # Mid[q] = midpoint of edge (q, q+1)
    C = np.zeros(2)
    quads = [np.stack([C, Mid[(q - 1) % sides], V[q], Mid[q]]) for q in range(sides)]
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.reshape(-1), j.reshape(-1), k.reshape(-1)
    rr, ss, tt = r1d[i], r1d[j], r1d[k]
    wts = np.stack([(1 - rr) * (1 - ss), (1 + rr) * (1 - ss), (1 + rr) * (1 + ss),
                    (1 - rr) * (1 + ss)], axis=1) / 4.0        # [n3, 4] bilinear weights
    xyz = []
    for layer in range(nz):
        z0, z1 = height * layer / nz, height * (layer + 1) / nz
        z = z0 + (1.0 + tt) / 2.0 * (z1 - z0)
        for P in quads:
            xy = wts @ P                                       # [n3, 2]
            xyz.append(np.stack([xy[:, 0], xy[:, 1], z], axis=0))
    xyz = np.ascontiguousarray(np.stack(xyz))                  # [E, 3, n3]
    E = xyz.shape[0]
    # global ids by coordinates
    key = np.round(xyz.transpose(0, 2, 1).reshape(-1, 3) / (1e-9 * radius)).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    inv = inv.reshape(-1)
    # ids in order of first appearance (element-major), coordinates from that copy
    order = np.argsort(first, kind="stable")
    rank_of = np.empty_like(order)
    rank_of[order] = np.arange(order.size)
    glo = rank_of[inv].reshape(E, n ** 3).astype(np.int64)
    flat = xyz.transpose(0, 2, 1).reshape(-1, 3)
    canon = flat[first[order]]
    xyz = np.ascontiguousarray(canon[glo.reshape(-1)].reshape(E, n ** 3, 3).transpose(0, 2, 1))
    # boundary faces: faces whose node set appears in one element only
    faces = []
    for axis, val in ((0, 0), (0, N), (1, 0), (1, N), (2, 0), (2, N)):
        sel = (i, j, k)[axis] == val
        faces.append(np.nonzero(sel)[0])
    count = {}
    fkeys = []
    for e in range(E):
        for f in faces:
            fk = tuple(sorted(glo[e, f].tolist()))
            fkeys.append((e, f, fk))
            count[fk] = count.get(fk, 0) + 1
    bnd = np.zeros(int(glo.max()) + 1, dtype=bool)
    for e, f, fk in fkeys:
        if count[fk] == 1:
            bnd[glo[e, f]] = True
    dirichlet = bnd[glo].astype(np.uint8)
    eidx = np.zeros((E, 3), dtype=np.int64)
    return Mesh(N=N, xyz=xyz, glo=np.ascontiguousarray(glo), dirichlet=np.ascontiguousarray(dirichlet),
                elems=(sides, 1, nz), lengths=(radius, radius, height), eidx=eidx)
