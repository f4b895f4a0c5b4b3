"""Multi-GPU domain decomposition of the assembly: z-slabs + interface sum.

The reference has no distributed path (the
assembly is "trivially parallel"); this is the B200 extension of its
element-slab parallelism (variants.py:467-503, _slab_bounds) to one process
per GPU.  The path shards naturally: rank r assembles the contiguous cell
layers [k_r, k_{r+1}) of a structured box, which are a contiguous element
range (e = 6 (i + nx (j + ny k)) + t, mesh.py:148-150) touching node planes
k_r .. k_{r+1}.  Only the two interface planes are shared, so the single
exchange step is: every rank sends its partial RHS of each interface plane
to the neighbour and adds what it receives (NCCL send/recv over NVLink,
``torch.distributed`` as the plumbing).  Each shared node then holds the full
sum on both ranks.

``SlabPartition`` is pure host logic (tested with gloo on CPU);
``SlabDomain`` binds it to an ``Assembler`` on the rank's GPU.

General (unstructured or renumbered) meshes: ``MeshPartition`` cuts the
elements by recursive coordinate bisection of their centroids (SURVEY.md
section 8e); a node may then be shared by several ranks and a rank may have
many neighbours, so ``PartitionedDomain`` sums with the NCCL exchange (each
rank sends its local partial of every node it shares with a neighbour, then
adds what it receives: every sharer ends with the full sum).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .mesh import Mesh, _box_arrays


def slab_bounds(n_layers: int, world: int) -> list[tuple[int, int]]:
    """Near-equal contiguous split (same rule as variants._slab_bounds)."""
    q, r = divmod(n_layers, world)
    out, lo = [], 0
    for i in range(world):
        hi = lo + q + (1 if i < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _axis(n: int, ext: float) -> np.ndarray:
    # np.linspace(0, ext, n+1) semantics (mesh.py:159-161)
    v = np.arange(n + 1, dtype=np.float64) * (ext / n)
    v[-1] = ext
    return v


@dataclass(frozen=True)
class SlabPartition:
    """Rank ``rank``'s z-slab of an (nx, ny, nz) Kuhn box over ``world`` ranks."""

    cells: tuple[int, int, int]
    rank: int
    world: int
    extents: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        nx, ny, nz = self.cells
        if nz < self.world:
            raise ValueError("need at least one cell layer per rank")
        if not 0 <= self.rank < self.world:
            raise ValueError("rank out of range")

    @property
    def layers(self) -> tuple[int, int]:
        return slab_bounds(self.cells[2], self.world)[self.rank]

    @property
    def plane(self) -> int:
        nx, ny, _ = self.cells
        return (nx + 1) * (ny + 1)

    @property
    def n_global_nodes(self) -> int:
        nx, ny, nz = self.cells
        return (nx + 1) * (ny + 1) * (nz + 1)

    @property
    def node_range(self) -> tuple[int, int]:
        """Global node ids [lo, hi) of this slab (node planes k0..k1)."""
        k0, k1 = self.layers
        return k0 * self.plane, (k1 + 1) * self.plane

    @property
    def elem_range(self) -> tuple[int, int]:
        nx, ny, _ = self.cells
        k0, k1 = self.layers
        return 6 * nx * ny * k0, 6 * nx * ny * k1

    def local_mesh(self) -> Mesh:
        """The slab as a mesh; local node l <-> global node node_range[0] + l,
        coordinates bitwise equal to the global box's."""
        nx, ny, nz = self.cells
        k0, k1 = self.layers
        _, conn = _box_arrays(nx, ny, k1 - k0)
        xs = _axis(nx, self.extents[0])
        ys = _axis(ny, self.extents[1])
        zs = _axis(nz, self.extents[2])[k0:k1 + 1]
        zz, yy, xx = np.meshgrid(zs, ys, xs, indexing="ij")
        coords = np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()])
        return Mesh(coords=coords, connectivity=conn)

    def interfaces(self) -> dict[int, np.ndarray]:
        """Neighbour rank -> local node ids of the shared plane (same global
        order on both sides)."""
        k0, k1 = self.layers
        P = self.plane
        out = {}
        if self.rank > 0:
            out[self.rank - 1] = np.arange(0, P, dtype=np.int64)
        if self.rank < self.world - 1:
            out[self.rank + 1] = np.arange((k1 - k0) * P, (k1 - k0 + 1) * P, dtype=np.int64)
        return out

    def owned_mask(self) -> np.ndarray:
        """Nodes this rank reports in a gathered global vector (the top plane
        belongs to the upper neighbour)."""
        lo, hi = self.node_range
        m = np.ones(hi - lo, dtype=bool)
        if self.rank < self.world - 1:
            m[-self.plane:] = False
        return m

    def velocity(self, spec: str, mesh: Optional[Mesh] = None) -> np.ndarray:
        """The global field restricted to this slab (global extents / rng)."""
        from .fields import make_velocity
        mesh = mesh or self.local_mesh()
        name, _, arg = spec.partition(":")
        lo, hi = self.node_range
        if name == "random":
            seed = int(arg) if arg else 0
            # draw the global stream, keep this slab's rows (bitwise the global field)
            rng = np.random.default_rng(seed)
            if lo:
                rng.uniform(-1.0, 1.0, size=(lo, 3))
            return rng.uniform(-1.0, 1.0, size=(hi - lo, 3))
        if name == "taylor-green":
            c = mesh.coords
            s = np.pi * c / np.asarray(self.extents)
            u = np.zeros((c.shape[0], 3))
            u[:, 0] = np.sin(s[:, 0]) * np.cos(s[:, 1]) * np.cos(s[:, 2])
            u[:, 1] = -np.cos(s[:, 0]) * np.sin(s[:, 1]) * np.cos(s[:, 2])
            return u
        return make_velocity(mesh, spec)


def rcb_parts(points: np.ndarray, world: int) -> np.ndarray:
    """Recursive coordinate bisection: a part id in [0, world) per point
    (native, csrc/tal_meshio.cpp: rcb_parts).

    Each level splits the current set along its largest extent (first axis
    on ties) at the count that gives the two halves floor(k/2) and ceil(k/2)
    of the k parts (balanced to one element); ties in the coordinate keep
    the set's order (a stable sort), so every rank computes the same
    partition.  Sub-problems of a level run in parallel on the host."""
    from ._native import check, lib, ptr
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if world < 1:
        raise ValueError("world must be >= 1")
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must have shape (n, 3)")
    part = np.zeros(pts.shape[0], dtype=np.int32)
    check(lib().tal_rcb_parts(ptr(pts), pts.shape[0], int(world), ptr(part)))
    return part


class MeshPartition:
    """Rank ``rank``'s share of a general mesh cut into ``world`` parts.

    ``parts`` (element -> rank) defaults to RCB of the element centroids.
    Local nodes are the rank's element nodes in ascending global id, so a
    shared node has the same relative order on every sharer; its owner (for
    a gathered global vector) is the lowest sharing rank."""

    def __init__(self, mesh, rank: int, world: int, parts: Optional[np.ndarray] = None):
        if not 0 <= rank < world:
            raise ValueError("rank out of range")
        self.rank, self.world = rank, world
        coords = np.asarray(mesh.coords, dtype=np.float64)
        conn = np.asarray(mesh.connectivity, dtype=np.int64)
        self.n_global_nodes = coords.shape[0]
        if parts is None:
            parts = rcb_parts(coords[conn].mean(axis=1), world)
        self.parts = np.asarray(parts, dtype=np.int32)
        if self.parts.shape != (conn.shape[0],) or (self.parts.size and (
                self.parts.min() < 0 or self.parts.max() >= world)):
            raise ValueError("parts must give a rank in [0, world) per element")
        mine = np.flatnonzero(self.parts == rank)
        self.elements = mine                                   # global element ids
        self.global_nodes = np.unique(conn[mine])              # local -> global node id
        self._coords = coords[self.global_nodes]
        self._conn = np.searchsorted(self.global_nodes, conn[mine])
        # (node, rank) incidence -> sharers of each of my nodes
        nv = np.unique(conn.ravel() * world + np.repeat(self.parts.astype(np.int64), 4))
        node, rk = nv // world, (nv % world).astype(np.int32)
        owner = np.full(self.n_global_nodes, world, dtype=np.int32)
        np.minimum.at(owner, node, rk)
        self._owner = owner[self.global_nodes]
        on_me = np.isin(node, self.global_nodes)
        self._ifaces = {}
        for nbr in np.unique(rk[on_me & (rk != rank)]):
            g = node[on_me & (rk == nbr)]                      # ascending global ids
            self._ifaces[int(nbr)] = np.searchsorted(self.global_nodes, g)

    def local_mesh(self) -> Mesh:
        return Mesh(coords=self._coords, connectivity=self._conn)

    def interfaces(self) -> dict[int, np.ndarray]:
        """Neighbour rank -> local ids of the nodes shared with it (ascending
        global id: the same order on both sides)."""
        return dict(self._ifaces)

    def owned_mask(self) -> np.ndarray:
        return self._owner == self.rank

    def velocity(self, u_global: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(u_global)[self.global_nodes])


def exchange_interfaces(part, send: dict, recv: dict, group=None) -> None:
    """Post the interface-plane send/recv pairs with every neighbour and wait.

    ``send[nbr]`` / ``recv[nbr]`` are same-shaped tensors (CUDA under NCCL, CPU
    under gloo); after return ``recv[nbr]`` holds the neighbour's partial sums.
    """
    import torch.distributed as dist
    ops = []
    for nbr in sorted(send):
        ops.append(dist.P2POp(dist.isend, send[nbr], nbr, group=group))
        ops.append(dist.P2POp(dist.irecv, recv[nbr], nbr, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class SlabDomain:
    """One rank's slab on its GPU: local assembly + the interface sum.

    ``fused`` (default for scatter='private-atomic'): the assembly kernel
    itself REDs the interface-plane partial sums into the neighbours' RHS over
    peer memory (CUDA IPC; include/tal_b200.h "fused interface sum") -- one
    launch per step plus four tiny flag kernels, no separate exchange.
    Otherwise: local assembly, then an NCCL send/recv of the interface planes
    and a halo-add kernel (``exchange_interfaces``).
    """

    def __init__(self, cells, rank: int, world: int, cfg=None, fused: Optional[bool] = None):
        import torch

        from .assembly import Assembler, RunConfig
        self.part = SlabPartition(tuple(int(c) for c in cells), rank, world)
        self.cfg = cfg or RunConfig()
        self.mesh = self.part.local_mesh()
        ifaces = self.part.interfaces()
        if fused is None:
            fused = self.cfg.scatter == "private-atomic" and world > 1
        self.fused = bool(fused) and bool(ifaces)
        ext = np.concatenate(list(ifaces.values())) if self.fused else None
        self.assembler = Assembler(self.mesh, self.cfg, external_nodes=ext)
        dev = torch.device("cuda", self.cfg.device)
        self._lists, self._send, self._recv = {}, {}, {}
        self.fused_error = None
        self._graph_params = None
        if self.fused:
            if self._connect_peers(ifaces):
                return
            # a rank could not map its neighbours' memory (no P2P / IPC on
            # this system): every rank switches to the NCCL exchange path;
            # the external (interface) nodes are REDed either way
            self.fused = False
        for nbr, ids in ifaces.items():
            internal = self.assembler.map_nodes(ids)
            self._lists[nbr] = torch.as_tensor(internal, device=dev)
            self._send[nbr] = torch.empty((ids.size, 3), dtype=torch.float64, device=dev)
            self._recv[nbr] = torch.empty((ids.size, 3), dtype=torch.float64, device=dev)

    def _connect_peers(self, ifaces) -> bool:
        """Exchange IPC handles and interface internal ids with the neighbours
        (host objects over torch.distributed), then open the peer mappings.
        Returns whether EVERY rank succeeded (a collective decision)."""
        import torch.distributed as dist
        asm = self.assembler
        rh, off, fh = asm.peer_export()
        mine = {nbr: asm.map_nodes(ids) for nbr, ids in ifaces.items()}
        info = [None] * self.part.world
        dist.all_gather_object(info, (rh, off, fh, asm.n_nodes, mine))
        ok = True
        try:
            for nbr, ids in ifaces.items():
                prh, poff, pfh, pn, pmap = info[nbr]
                slot = 0 if nbr < self.part.rank else 1
                asm.peer_open(slot, prh, poff, pfh, pn, ids, pmap[self.part.rank])
        except RuntimeError as err:
            ok, self.fused_error = False, str(err)
        votes = [None] * self.part.world
        dist.all_gather_object(votes, ok)
        if not all(votes):
            if ok:
                asm.peer_detach()
            return False
        dist.barrier()
        return True

    def velocity(self, spec: str) -> np.ndarray:
        u = self.part.velocity(spec, self.mesh)
        self.assembler.set_velocity_host(u, stream=0)
        return u

    def step(self, params, stream=0) -> int:
        """One assembly including the interface sum; returns kernels launched.
        Fused: the whole step (zeroing, flag signals/waits, kernel) is one
        captured CUDA graph, re-captured when ``params`` change."""
        asm = self.assembler
        if self.fused:
            if self._graph_params != params:
                asm.capture(params)
                self._graph_params = params
            return asm.replay(stream=stream)
        n = asm.run(params, stream=stream)
        for nbr, lst in self._lists.items():
            asm.halo_pack(lst.data_ptr(), lst.numel(), self._send[nbr].data_ptr(), stream=stream)
            n += 1
        if self._host_staged():  # gloo (validation runs): stage the planes through host memory
            send = {k: v.cpu() for k, v in self._send.items()}
            recv = {k: v.cpu() for k, v in self._recv.items()}
            exchange_interfaces(self.part, send, recv)
            for k, v in recv.items():
                self._recv[k].copy_(v)
        else:
            exchange_interfaces(self.part, self._send, self._recv)
        for nbr, lst in self._lists.items():
            asm.halo_accumulate(lst.data_ptr(), lst.numel(), self._recv[nbr].data_ptr(), stream=stream)
            n += 1
        return n

    @staticmethod
    def _host_staged() -> bool:
        import torch.distributed as dist
        return dist.is_initialized() and dist.get_backend() == "gloo"

    def owned_rhs(self) -> tuple[np.ndarray, np.ndarray]:
        """(global node ids, rhs rows) this rank reports after a step."""
        rhs = self.assembler.get_rhs_host(stream=0)
        self.assembler.synchronize(stream=0)
        mask = self.part.owned_mask()
        return self._global_ids()[mask], rhs[mask]

    def _global_ids(self) -> np.ndarray:
        lo, hi = self.part.node_range
        return np.arange(lo, hi, dtype=np.int64)

    def close(self) -> None:
        self.assembler.close()


class PartitionedDomain(SlabDomain):
    """One rank's part of a general mesh (``MeshPartition``) on its GPU: local
    assembly, then the NCCL exchange of the shared-node partial sums with
    every neighbour (``SlabDomain.step``'s exchange path).  The fused
    peer-memory sum needs the slab's at most two neighbours, so it is not
    used here."""

    def __init__(self, mesh, rank: int, world: int, cfg=None, parts: Optional[np.ndarray] = None):
        import torch

        from .assembly import Assembler, RunConfig
        self.part = MeshPartition(mesh, rank, world, parts)
        self.cfg = cfg or RunConfig()
        self.mesh = self.part.local_mesh()
        self.fused, self.fused_error, self._graph_params = False, None, None
        self.assembler = Assembler(self.mesh, self.cfg)
        dev = torch.device("cuda", self.cfg.device)
        self._lists, self._send, self._recv = {}, {}, {}
        for nbr, ids in self.part.interfaces().items():
            self._lists[nbr] = torch.as_tensor(self.assembler.map_nodes(ids), device=dev)
            self._send[nbr] = torch.empty((ids.size, 3), dtype=torch.float64, device=dev)
            self._recv[nbr] = torch.empty((ids.size, 3), dtype=torch.float64, device=dev)

    def set_velocity(self, u_global: np.ndarray) -> np.ndarray:
        u = self.part.velocity(u_global)
        self.assembler.set_velocity_host(u, stream=0)
        return u

    def _global_ids(self) -> np.ndarray:
        return self.part.global_nodes
