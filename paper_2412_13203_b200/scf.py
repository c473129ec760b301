"""Closed-shell RHF driver over the GPU Fock build.

The caller of the hot path: one-electron S, T, V (host), X = S^-1/2
(SPEC.md:464-472), core-Hamiltonian guess, Roothaan iterations with
F = H + 2J - K from ``Engine.build_jk`` (one GPU Fock build per iteration),
optional DIIS (depth 6), convergence on the max-abs density
change (default 1e-6) and max_iter 99 (§7.5).
E = sum D (H + F) + E_nuc with D = C_occ C_occ^T.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np


@dataclass
class ScfResult:
    energy: float
    iterations: int
    converged: bool
    energies: List[float] = field(default_factory=list)
    density: Optional[np.ndarray] = None
    fock_builds: int = 0
    tune_sweeps: int = 0  # Workload Allocator sweeps interleaved with the first iterations


def orthogonalizer(S: np.ndarray, tol: float = 1e-10) -> np.ndarray:
    """Symmetric X = S^-1/2; linear dependence is an error."""
    w, U = np.linalg.eigh(S)
    if w.min() < tol:
        raise np.linalg.LinAlgError(f"overlap has eigenvalue {w.min():.3e} < {tol:g} (linear dependence)")
    return (U * w ** -0.5) @ U.T


def density_from_mos(C: np.ndarray, nocc: int) -> np.ndarray:
    if nocc > C.shape[1]:
        raise ValueError("n_occ exceeds the basis dimension")
    Co = C[:, :nocc]
    return Co @ Co.T


def rhf(build_jk: Callable[[np.ndarray], tuple], S: np.ndarray, H: np.ndarray, e_nuc: float, nocc: int,
        conv: float = 1e-6, max_iter: int = 99, diis: bool = True, damping: float = 0.0,
        e_conv: float = 1e-10) -> ScfResult:
    """Roothaan/DIIS loop; ``build_jk(D) -> (J, K)`` is the Fock build."""
    X = orthogonalizer(S)
    _, Cp = np.linalg.eigh(X.T @ H @ X)
    D = density_from_mos(X @ Cp, nocc)
    res = ScfResult(energy=0.0, iterations=0, converged=False)
    focks, errs = [], []
    E_old = None
    for it in range(1, max_iter + 1):
        J, K = build_jk(D)
        res.fock_builds += 1
        F = H + 2.0 * J - K
        E = float(np.sum(D * (H + F)) + e_nuc)
        if not np.isfinite(E):
            raise FloatingPointError("SCF energy is not finite")
        res.energies.append(E)
        Fs = F
        if diis:
            err = X.T @ (F @ D @ S - S @ D @ F) @ X
            focks.append(F)
            errs.append(err)
            if len(focks) > 6:
                focks.pop(0)
                errs.pop(0)
            n = len(focks)
            if n >= 2:
                B = -np.ones((n + 1, n + 1))
                B[n, n] = 0.0
                for a in range(n):
                    for b in range(n):
                        B[a, b] = np.sum(errs[a] * errs[b])
                rhs = np.zeros(n + 1)
                rhs[n] = -1.0
                try:
                    c = np.linalg.solve(B, rhs)[:n]
                    Fs = sum(ci * Fi for ci, Fi in zip(c, focks))
                except np.linalg.LinAlgError:
                    Fs = F
        _, Cp = np.linalg.eigh(X.T @ Fs @ X)
        Dn = density_from_mos(X @ Cp, nocc)
        if damping > 0.0 and not diis:
            Dn = (1.0 - damping) * Dn + damping * D
        dD = float(np.max(np.abs(Dn - D)))
        D = Dn
        res.iterations = it
        if dD < conv and (E_old is not None and abs(E - E_old) < e_conv):
            res.converged = True
            break
        E_old = E
    # final energy with the converged density
    J, K = build_jk(D)
    res.fock_builds += 1
    F = H + 2.0 * J - K
    res.energy = float(np.sum(D * (H + F)) + e_nuc)
    res.density = D
    return res


def rhf_device(engine, S: np.ndarray, H: np.ndarray, e_nuc: float, nocc: int, conv: float = 1e-6,
               max_iter: int = 99, diis: bool = True, e_conv: float = 1e-10) -> ScfResult:
    """Device-resident Roothaan/DIIS loop: D, J, K, F and
    the DIIS history stay in HBM; the Fock build is ``build_jk_device`` on
    the current torch stream, the orthogonalised eigenproblem is
    ``torch.linalg.eigh`` (cuSOLVER syevd) and D = C_occ C_occ^T a DGEMM.
    Only the energy and the convergence scalars come back to the host."""
    import torch
    stream = torch.cuda.Stream()  # one explicit stream for torch ops and the Fock build
    with torch.cuda.stream(stream):
        return _rhf_device(engine, S, H, e_nuc, nocc, conv, max_iter, diis, e_conv, stream.cuda_stream)


def _rhf_device(engine, S, H, e_nuc, nocc, conv, max_iter, diis, e_conv, st) -> ScfResult:
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.as_tensor(a, dtype=torch.float64, device=dev).contiguous()
    Sd, Hd = t(S), t(H)
    X = t(orthogonalizer(S))
    N = Hd.shape[0]
    J = torch.empty((N, N), dtype=torch.float64, device=dev)
    K = torch.empty_like(J)

    def fock_build(D):
        engine.build_jk_device(D.data_ptr(), J.data_ptr(), K.data_ptr(), st)
        return J, K

    def density(F):
        _, Cp = torch.linalg.eigh(X.T @ F @ X)
        C = X @ Cp[:, :nocc]
        return C @ C.T

    D = density(Hd).contiguous()
    res = ScfResult(energy=0.0, iterations=0, converged=False)
    focks, errs = [], []
    E_old = None
    for it in range(1, max_iter + 1):
        J_, K_ = fock_build(D)
        res.fock_builds += 1
        F = Hd + 2.0 * J_ - K_
        E = float(torch.sum(D * (Hd + F))) + e_nuc
        if not np.isfinite(E):
            raise FloatingPointError("SCF energy is not finite")
        res.energies.append(E)
        Fs = F
        if diis:
            focks.append(F.clone())
            errs.append(X.T @ (F @ D @ Sd - Sd @ D @ F) @ X)
            if len(focks) > 6:
                focks.pop(0)
                errs.pop(0)
            n = len(focks)
            if n >= 2:
                E_ = torch.stack(errs).reshape(n, -1)
                B = -torch.ones((n + 1, n + 1), dtype=torch.float64, device=dev)
                B[n, n] = 0.0
                B[:n, :n] = E_ @ E_.T
                rhs = torch.zeros(n + 1, dtype=torch.float64, device=dev)
                rhs[n] = -1.0
                try:
                    c = torch.linalg.solve(B, rhs)[:n]
                    Fs = torch.einsum("i,ijk->jk", c, torch.stack(focks))
                except RuntimeError:
                    Fs = F
        Dn = density(Fs).contiguous()
        dD = float(torch.max(torch.abs(Dn - D)))
        D = Dn
        res.iterations = it
        if dD < conv and (E_old is not None and abs(E - E_old) < e_conv):
            res.converged = True
            break
        E_old = E
    J_, K_ = fock_build(D)
    res.fock_builds += 1
    F = Hd + 2.0 * J_ - K_
    res.energy = float(torch.sum(D * (Hd + F))) + e_nuc
    res.density = D.cpu().numpy()
    return res


def interleave_tuning(engine, build_jk: Callable[[np.ndarray], tuple], tune_variants: bool = True,
                      reps: int = 3):
    """Wrap a Fock build so the Workload Allocator runs inside the first SCF
    iterations on the live density ("integrates with ongoing
    computations at runtime"): the first build picks the kernel
    variant per class, then every build runs one Alg. 2 sweep (combine /
    measure / revert of the granularity) until a sweep finds no improvement.
    Tuning changes J/K only by atomic summation order. Returns (build, state)."""
    state = {"sweeps": 0, "converged": False, "variants": not tune_variants}

    def build(D):
        if not state["variants"]:
            engine.tune(D, reps=reps)
            state["variants"] = True
        if not state["converged"]:
            state["converged"] = not engine.tune_step(D, reps)
            state["sweeps"] += 1
        return build_jk(D)

    return build, state


def run_rhf(xyz_text: str, basis_text: str, tau: float = 1e-12, device: int = 0, kappa_screen: float = 0.0,
            device_resident: bool = False, tune: bool = False, **kw) -> ScfResult:
    """Full driver on one GPU: load, pairs, Schwarz, screening, SCF. With
    ``device_resident`` the post-Fock step runs on the GPU too (rhf_device).
    With ``tune`` the Workload Allocator is interleaved with the first
    iterations (interleave_tuning)."""
    from .eritile import Engine
    e = Engine(device).load_molecule(xyz_text, basis_text).build_pairs(kappa_screen)
    e.set_screening(tau)
    S, T, V = e.one_electron()
    if device_resident:
        import torch
        torch.cuda.set_device(device)
        return rhf_device(e, S, T + V, e.nuclear_repulsion(), e.nelectrons // 2, **kw)
    build = e.build_jk
    state = None
    if tune:
        build, state = interleave_tuning(e, e.build_jk)
    res = rhf(build, S, T + V, e.nuclear_repulsion(), e.nelectrons // 2, **kw)
    if state is not None:
        res.tune_sweeps = state["sweeps"]
    return res
