"""Symmetric block-sparse matrices (drop-in for `stiffbody.sparse`, sparse.py:1-174).

`BlockSparseMatrix` keeps the reference's host container semantics
(fixed pattern, upper off-diagonal storage, out-of-pattern adds raise).
`matvec` and `factor().solve*` run on the GPU: `factor()` is the device
sparse block Cholesky (kernel K4, csrc/k_chol.cu: minimum-degree order,
elimination-tree levels, refinement as solve_refined); `BlockJacobiPCG`
keeps the iterative alternative under the same 1e-8 relative residual
contract.  Blocks smaller than 12 are padded to 12 on the device.
"""
from __future__ import annotations

import warnings

import numpy as np

from . import _native

__all__ = ["BlockSparseMatrix", "BlockCholesky", "BlockJacobiPCG", "FactorizationError", "PcgNotConverged"]


class FactorizationError(RuntimeError):
    """Non-SPD diagonal block; `block` is its index (sparse.py:17-25)."""

    def __init__(self, block: int, message: str = ""):
        self.block = block
        super().__init__(message or f"non-SPD pivot at diagonal block {block} "
                         "(per-pair PSD projection violated?)")


class PcgNotConverged(RuntimeError):
    pass


class BlockSparseMatrix:
    def __init__(self, n_blocks: int, pairs=(), block_dim: int = 12):
        self.n = int(n_blocks)
        self.b = int(block_dim)
        self.diag = np.zeros((self.n, self.b, self.b))
        self.off: dict = {}
        for i, j in pairs:
            key = (min(int(i), int(j)), max(int(i), int(j)))
            if key[0] == key[1]:
                raise ValueError("off-diagonal pair must couple two blocks")
            if key not in self.off:
                self.off[key] = np.zeros((self.b, self.b))

    @property
    def shape(self):
        return (self.n * self.b, self.n * self.b)

    def reset(self):
        self.diag[:] = 0.0
        for blk in self.off.values():
            blk[:] = 0.0

    def add_diag(self, i: int, block: np.ndarray):
        self.diag[i] += block

    def add_off(self, i: int, j: int, block: np.ndarray):
        if i < j:
            self.off[(i, j)] += block
        else:
            self.off[(j, i)] += np.asarray(block).T

    def to_dense(self) -> np.ndarray:
        b = self.b
        A = np.zeros(self.shape)
        for i in range(self.n):
            A[i * b:(i + 1) * b, i * b:(i + 1) * b] = self.diag[i]
        for (i, j), blk in self.off.items():
            A[i * b:(i + 1) * b, j * b:(j + 1) * b] = blk
            A[j * b:(j + 1) * b, i * b:(i + 1) * b] = blk.T
        return A

    def _packed(self):
        keys = sorted(self.off.keys())
        k = np.array(keys, dtype=np.int64).reshape(-1, 2)
        off = (np.array([self.off[x] for x in keys]).reshape(-1, self.b, self.b) if keys
               else np.zeros((0, self.b, self.b)))
        return k, off

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """y = A x on the GPU BSR SpMV (sparse.py:77-84)."""
        k, off = self._packed()
        return _native.bsr_matvec(self.n, self.b, self.diag, k, off, np.asarray(x, dtype=float))

    def factor(self) -> "BlockCholesky":
        return BlockCholesky(self)


class BlockCholesky:
    """L L^T = A on the GPU (sparse.py:87-161).

    Construction factors once (raising FactorizationError(block) on a non-SPD
    pivot); the solves re-run the device factor + triangular solves on the
    current contents of A (the container is host-side and mutable).
    """

    def __init__(self, A: BlockSparseMatrix):
        self._A = A
        self.last_solves = 0
        self.last_rel_residual = 0.0
        if A.n:
            k, off = A._packed()
            _native.bsr_cholesky(A.n, A.b, A.diag, k, off, np.zeros(A.n * A.b), 0.0, 0)

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        """One forward/backward substitution (sparse.py:131-147)."""
        return self.solve_refined(rhs, rel_tol=0.0, max_refine=0)

    def solve_refined(self, rhs: np.ndarray, rel_tol: float = 1e-8, max_refine: int = 3) -> np.ndarray:
        """Iterative refinement until |A x - rhs| <= rel_tol |rhs| (sparse.py:149-161)."""
        A = self._A
        rhs = np.asarray(rhs, dtype=float).reshape(-1)
        if A.n == 0:
            return np.zeros(0)
        k, off = A._packed()
        x, ns, rel = _native.bsr_cholesky(A.n, A.b, A.diag, k, off, rhs, rel_tol, max_refine)
        self.last_solves, self.last_rel_residual = ns, rel
        return x


class BlockJacobiPCG:
    """Solver object standing in for BlockCholesky (same solve/solve_refined API).

    Construction validates the block-Jacobi preconditioner on the GPU, raising
    FactorizationError(block) for the first non-SPD diagonal block.
    """

    def __init__(self, A: BlockSparseMatrix):
        self._A = A
        self.last_iterations = 0
        self.last_rel_residual = 0.0
        if A.n:
            # probe the preconditioner (and the matrix) with a zero-cost solve of 0
            k, off = A._packed()
            _native.bsr_pcg(A.n, A.b, A.diag, k, off, np.zeros(A.n * A.b), 1e-8, 1)

    def solve_refined(self, rhs: np.ndarray, rel_tol: float = 1e-8, max_refine: int = 3,
                      max_iters: int = 200000) -> np.ndarray:
        A = self._A
        rhs = np.asarray(rhs, dtype=float).reshape(-1)
        if A.n == 0:
            return np.zeros(0)
        k, off = A._packed()
        x, it, rel = _native.bsr_pcg(A.n, A.b, A.diag, k, off, rhs, rel_tol, max_iters)
        self.last_iterations, self.last_rel_residual = it, rel
        if rel > rel_tol and rel_tol >= 1e-12:
            warnings.warn(f"block-Jacobi PCG stopped at relative residual {rel:.3e} > {rel_tol:.1e}",
                          RuntimeWarning, stacklevel=2)
        return x

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        """Near machine-precision solve (the direct-solver contract of BlockCholesky.solve)."""
        return self.solve_refined(rhs, rel_tol=1e-14, max_iters=20000)
