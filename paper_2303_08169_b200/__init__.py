"""B200-native Allegro-Legato NNQMD hot path: a thin ctypes binding of include/allegro.h.

Argument marshalling only -- every step of the method (neighbour build, model,
forces, Verlet, outliers) runs in the CUDA kernels of ``libpaper_allegro.so``.
Importing this package requires the in-tree library; there is no CPU fallback.

Names follow the C ABI: ``allegro_create`` -> ``Allegro(...)``,
``allegro_compute_energy_forces`` -> ``Allegro.compute_energy_forces``,
``md_set_state`` / ``md_step`` / ``md_get_state`` / ``md_count_outliers`` /
``md_force_baseline`` -> methods of the same names.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALLEGRO_LIB") or os.path.join(_HERE, "lib", "libpaper_allegro.so")  # override: A/B builds

OK = 0
E_ARG, E_GEOMETRY, E_NONFINITE, E_WEIGHTS, E_CUDA, E_NCCL, E_OOM, E_STATE = -1, -2, -3, -4, -5, -6, -7, -8
HOST, DEVICE = 0, 1
PREC_FP32, PREC_3XTF32, PREC_BF16X3, PREC_TF32, PREC_BF16 = 0, 1, 2, 3, 4

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2303_08169_b200/build.py` "
        "(there is no CPU fallback for the CUDA path)"
    )
_lib = C.CDLL(LIB_PATH)


class AllegroParams(C.Structure):
    _fields_ = [
        ("weights_path", C.c_char_p),
        ("r_cut", C.c_double),
        ("skin", C.c_double),
        ("box", C.c_double * 3),
        ("n_atoms_global", C.c_int64),
        ("device", C.c_int),
        ("rank", C.c_int),
        ("world_size", C.c_int),
        ("nccl_unique_id", C.c_void_p),
        ("grid", C.c_int * 3),
        ("precision", C.c_int),
        ("cuda_stream", C.c_void_p),
    ]


class MdReport(C.Structure):
    _fields_ = [
        ("steps_done", C.c_int64),
        ("e_pot", C.c_double),
        ("e_kin", C.c_double),
        ("e_total", C.c_double),
        ("temperature", C.c_double),
        ("n_outliers_last", C.c_int64),
        ("n_edges", C.c_int64),
        ("n_rebuilds", C.c_int64),
        ("n_local", C.c_int64),
        ("xi", C.c_double),
        ("e_conserved", C.c_double),
    ]


class TtfProtocol(C.Structure):
    _fields_ = [
        ("nvt_steps", C.c_int64),
        ("T_K", C.c_double),
        ("tau_fs", C.c_double),
        ("max_nve_steps", C.c_int64),
        ("check_interval", C.c_int64),
        ("drift_tol", C.c_double),
        ("disp_max", C.c_double),
        ("outlier_k", C.c_double),
        ("outlier_interval", C.c_int64),
    ]


class TtfResult(C.Structure):
    _fields_ = [
        ("steps_survived", C.c_int64),
        ("fail_step", C.c_int64),
        ("reason", C.c_int),
        ("failed_in_nvt", C.c_int),
        ("e0", C.c_double),
        ("e_last", C.c_double),
        ("f_mean", C.c_double),
        ("f_sigma", C.c_double),
        ("n_series", C.c_int64),
    ]


class PimdReport(C.Structure):
    _fields_ = [
        ("steps_done", C.c_int64),
        ("e_pot_mean", C.c_double),
        ("e_spring", C.c_double),
        ("e_kin", C.c_double),
        ("h_conserved", C.c_double),
        ("temperature_beads", C.c_double),
        ("omega_p", C.c_double),
        ("n_edges", C.c_int64),
    ]


TTF_REASONS = {0: "censored", 1: "non_finite", 2: "displacement_blowup", 3: "energy_drift"}

_P = C.c_void_p
_lib.allegro_create.argtypes = [C.POINTER(AllegroParams), C.POINTER(_P)]
_lib.allegro_destroy.argtypes = [_P]
_lib.allegro_destroy.restype = None
_lib.allegro_last_error.argtypes = [_P]
_lib.allegro_last_error.restype = C.c_char_p
_lib.allegro_compute_energy_forces.argtypes = [_P, C.c_int64, C.c_int, _P, _P, _P, _P, _P, _P, _P]
_lib.md_set_state.argtypes = [_P, C.c_int64, _P, _P, _P]
_lib.md_get_state.argtypes = [_P, C.c_int64, _P, _P, _P]
_lib.md_step.argtypes = [_P, C.c_int64, C.c_double, C.POINTER(MdReport)]
_lib.md_count_outliers.argtypes = [_P, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int64)]
_lib.md_force_baseline.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
_lib.allegro_get_edges.argtypes = [_P, C.c_int64, C.POINTER(C.c_int64), _P, _P, _P]
_lib.allegro_get_edge_grad.argtypes = [_P, C.c_int64, _P]
_lib.allegro_get_row_edges.argtypes = [_P, C.c_int64, _P, C.c_int64, C.POINTER(C.c_int64), _P, _P, _P, _P]
_lib.allegro_chunk_starts.argtypes = [_P, C.c_int64, C.POINTER(C.c_int64), _P]
_lib.allegro_w3j_table.argtypes = [C.c_int, C.c_int, C.c_int, _P]
_lib.allegro_param_count.argtypes = [C.c_int, C.c_int]
_lib.allegro_param_count.restype = C.c_int64
_lib.allegro_layer_paths.argtypes = [C.c_int, C.c_int, _P]
_lib.allegro_version.restype = C.c_char_p
_lib.allegro_work_per_edge.argtypes = [C.c_int, C.c_int, _P]
_lib.md_step_host.argtypes = [_P, C.c_int64, C.c_int64, _P, _P, _P, _P, C.c_int64, C.c_double, C.POINTER(MdReport)]
_lib.allegro_profile.argtypes = [_P, C.c_int]
_lib.allegro_profile_read.argtypes = [_P, C.c_int, _P, _P, _P, _P]
_lib.allegro_launch_count.argtypes = [_P]
_lib.allegro_launch_count.restype = C.c_int64
_lib.allegro_profile_kind_name.argtypes = [C.c_int]
_lib.allegro_profile_kind_name.restype = C.c_char_p
_lib.allegro_nccl_unique_id.argtypes = [_P]
_lib.allegro_local_count.argtypes = [_P]
_lib.allegro_local_count.restype = C.c_int64
_lib.allegro_profile_detail.argtypes = [_P, C.c_int, _P, C.c_int, _P, _P, _P]
_lib.md_set_thermostat.argtypes = [_P, C.c_double, C.c_double]
_lib.allegro_compute_energy_forces_batch.argtypes = [_P, C.c_int64, C.c_int64, C.c_int, _P, _P, _P, _P, _P]
_lib.pimd_set_state.argtypes = [_P, C.c_int64, C.c_int64, _P, _P, _P, C.c_double]
_lib.pimd_step.argtypes = [_P, C.c_int64, C.c_double, C.POINTER(PimdReport)]
_lib.pimd_get_state.argtypes = [_P, _P, _P, _P, _P]
_lib.md_run_ttf.argtypes = [_P, C.c_double, C.POINTER(TtfProtocol), _P, C.c_int64, C.POINTER(TtfResult)]
_lib.md_get_local_state.argtypes = [_P, C.c_int64, C.POINTER(C.c_int64), _P, _P, _P, _P, _P]
_lib.allegro_debug_gemm.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, _P, _P, _P]
_lib.allegro_debug_gemm_epi.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P]
_lib.allegro_debug_gemm_bench.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_int, C.POINTER(C.c_double)]

EXPORTED = [
    "allegro_create", "allegro_destroy", "allegro_last_error", "allegro_compute_energy_forces",
    "md_set_state", "md_get_state", "md_step", "md_count_outliers", "md_force_baseline",
    "allegro_get_edges", "allegro_get_edge_grad", "allegro_w3j_table", "allegro_param_count",
    "allegro_layer_paths", "allegro_version", "md_step_host", "allegro_profile", "allegro_profile_read",
    "allegro_launch_count", "allegro_profile_kinds", "allegro_profile_kind_name", "allegro_debug_gemm",
    "allegro_debug_gemm_bench", "allegro_debug_gemm_epi", "allegro_nccl_unique_id", "allegro_local_count",
    "md_get_local_state", "md_set_thermostat", "md_run_ttf",
    "allegro_compute_energy_forces_batch", "pimd_set_state", "pimd_step", "pimd_get_state",
    "allegro_profile_detail", "allegro_work_per_edge", "allegro_get_row_edges", "allegro_chunk_starts",
]


class AllegroError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr(a) -> int | None:
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def w3j_table(l1: int, l2: int, l3: int) -> np.ndarray:
    out = np.zeros((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1))
    rc = _lib.allegro_w3j_table(l1, l2, l3, out.ctypes.data)
    if rc != OK:
        raise AllegroError(rc, "bad (l1, l2, l3)")
    return out.reshape(2 * l1 + 1, 2 * l2 + 1, 2 * l3 + 1)


def param_count(n_layers: int, lmax: int) -> int:
    return int(_lib.allegro_param_count(n_layers, lmax))


def layer_paths(n_layers: int, lmax: int):
    out = np.zeros(2 * n_layers, dtype=np.int32)
    _lib.allegro_layer_paths(n_layers, lmax, out.ctypes.data)
    return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(n_layers)]


def work_per_edge(n_layers: int, lmax: int):
    """(forward GEMM MACs, forward TP FMAs) per edge of the (n_layers, lmax) model."""
    out = np.zeros(2)
    rc = _lib.allegro_work_per_edge(n_layers, lmax, out.ctypes.data)
    if rc != OK:
        raise AllegroError(rc, "bad (n_layers, lmax)")
    return float(out[0]), float(out[1])


def debug_gemm(A: np.ndarray, W: np.ndarray, precision: int = PREC_FP32, device: int = 0) -> np.ndarray:
    """Test hook: C = A W with the library's contraction kernel (fp32 arrays)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float32)
    C_ = np.empty((A.shape[0], W.shape[1]), dtype=np.float32)
    rc = _lib.allegro_debug_gemm(device, precision, A.shape[0], W.shape[1], A.shape[1], A.ctypes.data,
                                 W.ctypes.data, C_.ctypes.data)
    if rc != OK:
        raise AllegroError(rc, _lib.allegro_last_error(None).decode())
    return C_


def debug_gemm_epi(A, W, epi, X=None, u=None, C=None, precision=PREC_3XTF32, want_aux=False, device=0):
    """Test hook: C = epi(0.75 * A W) with the optional X / u inputs; returns (C, aux)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float32)
    M, K = A.shape
    N = W.shape[1]
    Cv = np.zeros((M, N), np.float32) if C is None else np.ascontiguousarray(C, dtype=np.float32).copy()
    aux = np.zeros((M, N), np.float32) if want_aux else None
    Xv = None if X is None else np.ascontiguousarray(X, dtype=np.float32)
    uv = None if u is None else np.ascontiguousarray(u, dtype=np.float32)
    rc = _lib.allegro_debug_gemm_epi(device, precision, M, N, K, epi, A.ctypes.data, W.ctypes.data, _ptr(Xv), _ptr(uv),
                                     Cv.ctypes.data, _ptr(aux))
    if rc != OK:
        raise AllegroError(rc, _lib.allegro_last_error(None).decode())
    return Cv, aux


def debug_gemm_bench(M, N, K, epi=0, precision=PREC_3XTF32, iters=10, tma_store=1, max_stages=4, diag=0,
                     device=0) -> float:
    """Test hook: ms per launch of one contraction shape (device buffers, CUDA events)."""
    ms = C.c_double(0)
    rc = _lib.allegro_debug_gemm_bench(device, precision, M, N, K, epi, iters, tma_store, max_stages, diag, C.byref(ms))
    if rc != OK:
        raise AllegroError(rc, _lib.allegro_last_error(None).decode())
    return ms.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to every rank)."""
    buf = (C.c_char * 128)()
    rc = _lib.allegro_nccl_unique_id(C.addressof(buf))
    if rc != OK:
        raise AllegroError(rc, _lib.allegro_last_error(None).decode())
    return bytes(buf)


def version() -> str:
    return _lib.allegro_version().decode()


class Allegro:
    """One ctx of the C ABI (allegro_create ... allegro_destroy)."""

    def __init__(self, weights_path: str, box, r_cut: float = 0.0, skin: float = 0.0, device: int = 0,
                 n_atoms: int = 0, precision: int = PREC_3XTF32, stream: int | None = None, rank: int = 0,
                 world_size: int = 1, nccl_id: bytes | None = None, grid=(0, 0, 0)):
        p = AllegroParams()
        p.weights_path = os.fsencode(weights_path)
        p.r_cut = r_cut
        p.skin = skin
        for d in range(3):
            p.box[d] = float(box[d])
        p.n_atoms_global = n_atoms
        p.device = device
        p.rank, p.world_size = rank, world_size
        self._id = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        p.nccl_unique_id = None if self._id is None else C.addressof(self._id)
        for d in range(3):
            p.grid[d] = int(grid[d])
        p.precision = precision
        p.cuda_stream = stream
        h = _P()
        rc = _lib.allegro_create(C.byref(p), C.byref(h))
        if rc != OK:
            raise AllegroError(rc, _lib.allegro_last_error(None).decode())
        self._h = h
        self.box = np.asarray(box, dtype=np.float64)

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.allegro_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != OK:
            raise AllegroError(rc, _lib.allegro_last_error(self._h).decode())

    # ---- allegro_compute_energy_forces -------------------------------------------------
    def compute_energy_forces(self, pos, species, gid=None, box=None, e_atom=None, forces=None):
        """pos [n,3] f64, species [n] i32 (numpy => host pointers; torch cuda => device
        pointers, zero copy).  Returns (e_total, e_atom, forces) in the same kind.

        Device tensors are read and written on the ctx's stream (include/allegro.h): the
        caller's current torch stream is synchronised first, so the inputs are complete and
        the output blocks are no longer in use there; the call synchronises its own stream
        before it returns, so the outputs are complete afterwards."""
        n = int(pos.shape[0])
        on_dev = not isinstance(pos, np.ndarray)
        if on_dev:
            import torch

            assert pos.is_cuda and pos.dtype == torch.float64 and pos.is_contiguous()
            assert species.dtype == torch.int32 and species.is_contiguous()
            if e_atom is None:
                e_atom = torch.empty(n, dtype=torch.float64, device=pos.device)
            if forces is None:
                forces = torch.empty((n, 3), dtype=torch.float64, device=pos.device)
            torch.cuda.current_stream(pos.device).synchronize()
        else:
            pos = np.ascontiguousarray(pos, dtype=np.float64)
            species = np.ascontiguousarray(species, dtype=np.int32)
            gid = None if gid is None else np.ascontiguousarray(gid, dtype=np.int32)
            if e_atom is None:
                e_atom = np.empty(n, dtype=np.float64)
            if forces is None:
                forces = np.empty((n, 3), dtype=np.float64)
        bx = None if box is None else np.ascontiguousarray(box, dtype=np.float64)
        e = C.c_double(0.0)
        rc = _lib.allegro_compute_energy_forces(
            self._h, n, DEVICE if on_dev else HOST, _ptr(gid), _ptr(species), _ptr(pos),
            None if bx is None else bx.ctypes.data, C.addressof(e), _ptr(e_atom), _ptr(forces))
        self._check(rc)
        return e.value, e_atom, forces

    # ---- MD ---------------------------------------------------------------------------
    def md_set_state(self, species, pos, vel):
        species = np.ascontiguousarray(species, dtype=np.int32)
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        vel = np.ascontiguousarray(vel, dtype=np.float64)
        self.n = int(pos.shape[0])
        self._check(_lib.md_set_state(self._h, self.n, species.ctypes.data, pos.ctypes.data, vel.ctypes.data))

    def local_count(self) -> int:
        return int(_lib.allegro_local_count(self._h))

    def md_get_local_state(self, capacity: int | None = None):
        """This rank's owned atoms: (species, gid, pos, vel, forces) numpy arrays of length
        `capacity` (default: the local count); the first n_local rows are valid."""
        cap = self.local_count() if capacity is None else int(capacity)
        spc = np.zeros(cap, dtype=np.int32)
        gid = np.zeros(cap, dtype=np.int32)
        pos, vel, frc = np.zeros((cap, 3)), np.zeros((cap, 3)), np.zeros((cap, 3))
        n = C.c_int64(0)
        self._check(_lib.md_get_local_state(self._h, cap, C.byref(n), spc.ctypes.data, gid.ctypes.data,
                                            pos.ctypes.data, vel.ctypes.data, frc.ctypes.data))
        return n.value, spc, gid, pos, vel, frc

    def md_get_state(self):
        pos = np.empty((self.n, 3))
        vel = np.empty((self.n, 3))
        frc = np.empty((self.n, 3))
        self._check(_lib.md_get_state(self._h, self.n, pos.ctypes.data, vel.ctypes.data, frc.ctypes.data))
        return pos, vel, frc

    def md_step(self, n_steps: int, dt_fs: float = 2.0) -> MdReport:
        r = MdReport()
        self._check(_lib.md_step(self._h, n_steps, dt_fs, C.byref(r)))
        return r

    def md_set_thermostat(self, T_target: float = 200.0, tau_fs: float = 100.0):
        """Nose-Hoover NVT at T_target (K) with time constant tau_fs; tau_fs <= 0 -> NVE."""
        self._check(_lib.md_set_thermostat(self._h, T_target, tau_fs))

    def md_run_ttf(self, dt_fs: float = 2.0, nvt_steps: int = 1000, T_K: float = 200.0, tau_fs: float = 100.0,
                   max_nve_steps: int = 100000, check_interval: int = 100, drift_tol: float = 0.1,
                   disp_max: float = 0.5, outlier_k: float = 5.0, outlier_interval: int = 1):
        """Time-to-failure protocol (include/allegro.h md_run_ttf): NVT thermalisation, then NVE
        until non-finite / displacement blow-up / energy drift.  Returns (result dict, outlier
        series as an int64 array)."""
        pr = TtfProtocol(nvt_steps, T_K, tau_fs, max_nve_steps, check_interval, drift_tol, disp_max, outlier_k,
                         outlier_interval)
        cap = max(max_nve_steps, 0) // max(outlier_interval, 1)  # the C side validates the protocol
        series = np.zeros(max(cap, 1), dtype=np.int64)
        r = TtfResult()
        self._check(_lib.md_run_ttf(self._h, dt_fs, C.byref(pr), series.ctypes.data, cap, C.byref(r)))
        out = {f: getattr(r, f) for f, _ in TtfResult._fields_}
        out["reason_name"] = TTF_REASONS[r.reason]
        return out, series[: r.n_series].copy()

    def compute_energy_forces_batch(self, pos, species):
        """Replica batch (allegro_compute_energy_forces_batch): pos [n_rep][n_per][3], species
        [n_per] (host numpy) -> (e_rep [n_rep], e_atom [n_rep][n_per], forces [n_rep][n_per][3])."""
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        species = np.ascontiguousarray(species, dtype=np.int32)
        n_rep, n_per = pos.shape[0], pos.shape[1]
        e_rep = np.empty(n_rep)
        e_atom = np.empty((n_rep, n_per))
        frc = np.empty((n_rep, n_per, 3))
        self._check(_lib.allegro_compute_energy_forces_batch(self._h, n_rep, n_per, HOST, species.ctypes.data,
                                                             pos.ctypes.data, e_rep.ctypes.data, e_atom.ctypes.data,
                                                             frc.ctypes.data))
        return e_rep, e_atom, frc

    def pimd_set_state(self, species, pos, vel, T_K: float):
        """Ring-polymer state: species [n_per], pos / vel [n_beads][n_per][3] (host)."""
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        vel = np.ascontiguousarray(vel, dtype=np.float64)
        species = np.ascontiguousarray(species, dtype=np.int32)
        self._pimd_shape = pos.shape
        self._check(_lib.pimd_set_state(self._h, pos.shape[0], pos.shape[1], species.ctypes.data, pos.ctypes.data,
                                        vel.ctypes.data, T_K))

    def pimd_step(self, n_steps: int, dt_fs: float = 0.5) -> PimdReport:
        r = PimdReport()
        self._check(_lib.pimd_step(self._h, n_steps, dt_fs, C.byref(r)))
        return r

    def pimd_get_state(self):
        """-> (pos (unwrapped), vel, forces) [n_beads][n_per][3] and e_rep [n_beads]."""
        P, N, _ = self._pimd_shape
        pos, vel, frc, e = np.empty((P, N, 3)), np.empty((P, N, 3)), np.empty((P, N, 3)), np.empty(P)
        self._check(_lib.pimd_get_state(self._h, pos.ctypes.data, vel.ctypes.data, frc.ctypes.data, e.ctypes.data))
        return pos, vel, frc, e

    def md_count_outliers(self, mean: float, sigma: float, k: float = 5.0) -> int:
        c = C.c_int64(0)
        self._check(_lib.md_count_outliers(self._h, mean, sigma, k, C.byref(c)))
        return c.value

    def md_force_baseline(self):
        m, s = C.c_double(0), C.c_double(0)
        self._check(_lib.md_force_baseline(self._h, C.byref(m), C.byref(s)))
        return m.value, s.value

    def md_step_host(self, species, pos, vel, forces, n_steps: int = 1, dt_fs: float = 2.0,
                     n_local: int | None = None) -> MdReport:
        """End-to-end step on HOST arrays (updated in place): H2D, n_steps, D2H.
        numpy or (pinned) torch CPU tensors; their row count is the capacity passed to the C ABI."""
        r = MdReport()
        n = self.local_count() if n_local is None else int(n_local)
        cap = min(int(species.shape[0]), int(pos.shape[0]), int(vel.shape[0]), int(forces.shape[0]))
        self._check(_lib.md_step_host(self._h, n, cap, _ptr(species), _ptr(pos), _ptr(vel), _ptr(forces),
                                      n_steps, dt_fs, C.byref(r)))
        return r

    # ---- profiling -----------------------------------------------------------------
    def profile(self, enable: bool = True):
        self._check(_lib.allegro_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """{kind name: (time_ms, algorithmic flops, algorithmic bytes, launches)}"""
        out = {}
        for k in range(_lib.allegro_profile_kinds()):
            ms, fl, by, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
            self._check(_lib.allegro_profile_read(self._h, k, C.byref(ms), C.byref(fl), C.byref(by), C.byref(n)))
            out[_lib.allegro_profile_kind_name(k).decode()] = (ms.value, fl.value, by.value, n.value)
        return out

    def profile_detail(self):
        """[(shape tag, time_ms, algorithmic bytes, launches)] of tagged launches."""
        out = []
        k = 0
        while True:
            name = C.create_string_buffer(128)
            ms, by, n = C.c_double(), C.c_double(), C.c_int64()
            if _lib.allegro_profile_detail(self._h, k, name, 128, C.byref(ms), C.byref(by), C.byref(n)) != OK:
                break
            out.append((name.value.decode(), ms.value, by.value, n.value))
            k += 1
        return out

    def launch_count(self) -> int:
        return int(_lib.allegro_launch_count(self._h))

    # ---- test hooks -------------------------------------------------------------------
    def get_edges(self):
        n = C.c_int64(0)
        self._check(_lib.allegro_get_edges(self._h, 0, C.byref(n), None, None, None))
        E = n.value
        i = np.empty(E, dtype=np.int32)
        j = np.empty(E, dtype=np.int32)
        s = np.empty((E, 3), dtype=np.int8)
        self._check(_lib.allegro_get_edges(self._h, E, C.byref(n), i.ctypes.data, j.ctypes.data, s.ctypes.data))
        return i, j, s

    def get_row_edges(self, rows):
        """Edges of the listed owned rows: (i_gid, j_gid, shift [E][3], g [E][3])."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n = C.c_int64(0)
        self._check(_lib.allegro_get_row_edges(self._h, rows.size, rows.ctypes.data, 0, C.byref(n), None, None, None,
                                               None))
        E = n.value
        i = np.empty(E, dtype=np.int32)
        j = np.empty(E, dtype=np.int32)
        s = np.empty((E, 3), dtype=np.int8)
        g = np.empty((E, 3))
        self._check(_lib.allegro_get_row_edges(self._h, rows.size, rows.ctypes.data, E, C.byref(n), i.ctypes.data,
                                               j.ctypes.data, s.ctypes.data, g.ctypes.data))
        return i, j, s, g

    def chunk_starts(self):
        n = C.c_int64(0)
        self._check(_lib.allegro_chunk_starts(self._h, 0, C.byref(n), None))
        out = np.empty(max(n.value, 1), dtype=np.int64)
        self._check(_lib.allegro_chunk_starts(self._h, out.size, C.byref(n), out.ctypes.data))
        return out[: n.value]

    def get_edge_grad(self):
        n = C.c_int64(0)
        self._check(_lib.allegro_get_edges(self._h, 0, C.byref(n), None, None, None))
        g = np.empty((n.value, 3))
        self._check(_lib.allegro_get_edge_grad(self._h, n.value, g.ctypes.data))
        return g
