"""Thin ctypes binding of libdbfft.so (include/dbfft.h).  Argument marshalling only: every
step of the hot path runs in the CUDA kernels of csrc/.  torch provides device memory and
streams.  There is no CPU fallback: if the extension is missing this module raises."""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdbfft.so")

# ---------------------------------------------------------------------------- C types


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Env(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("cuda_stream", ctypes.c_void_p), ("device", ctypes.c_int32), ("loopback", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN),
                ("alloc_user", ctypes.c_void_p), ("pencil_rows", ctypes.c_int32)]


def torch_allocator(device):
    """dbfft_env allocator hooks backed by torch's CUDA caching allocator (the ctx's buffers show up
    in torch.cuda.memory_allocated and are recycled by torch after close())."""
    import torch

    def alloc(nbytes, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device)
        except Exception:  # noqa: BLE001  (out of memory -> NULL -> DBFFT_E_OOM)
            return None

    def free(ptr, _user):
        try:
            torch.cuda.caching_allocator_delete(ptr)
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    return ALLOC_FN(alloc), FREE_FN(free)

TRANSPORTS = {"nccl": 0, "peer": 1}


class Material(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("p", ctypes.c_double * 36)]


class Opts(ctypes.Structure):
    _fields_ = [("tol_eq", ctypes.c_double), ("tol_load", ctypes.c_double), ("tol_newton", ctypes.c_double),
                ("max_cg", ctypes.c_int32), ("max_newton", ctypes.c_int32), ("check_every", ctypes.c_int32),
                ("precond_refresh", ctypes.c_int32), ("precond_period", ctypes.c_int32),
                ("precond_medium", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("newton_iters", ctypes.c_int32),
                ("status", ctypes.c_int32), ("eps_eq", ctypes.c_double), ("eps_load", ctypes.c_double),
                ("max_dgrad", ctypes.c_double), ("macro_strain", ctypes.c_double * 9),
                ("macro_stress", ctypes.c_double * 9), ("bad_voxel", ctypes.c_int64), ("seconds", ctypes.c_double)]


MAT_ISO, MAT_CUBIC, MAT_NEOHOOKE, MAT_J2, MAT_SVK = 1, 2, 3, 4, 5
FIELD_U, FIELD_STRAIN, FIELD_STRESS, FIELD_U_HAT, FIELD_TANGENT = 0, 1, 2, 3, 4
STATUS = {0: "OK", 1: "E_INVALID_GRID", 2: "E_INVALID_ARG", 3: "E_STATE", 4: "E_CUDA", 5: "E_NCCL", 6: "E_OOM",
          7: "E_NOT_CONVERGED", 8: "E_BREAKDOWN", 9: "E_MATERIAL"}

# every symbol declared in include/dbfft.h
EXPORTS = ["dbfft_create", "dbfft_destroy", "dbfft_last_error", "dbfft_spectral_layout", "dbfft_set_phases",
           "dbfft_apply_K", "dbfft_apply_K_aug", "dbfft_precond", "dbfft_eval_state", "dbfft_default_opts",
           "dbfft_solve_increment", "dbfft_get_field", "dbfft_profile_enable", "dbfft_profile_read",
           "dbfft_profile_name", "dbfft_profile_count", "dbfft_launch_count", "dbfft_nccl_unique_id",
           "dbfft_residuals", "dbfft_incompatibility", "dbfft_get_trace", "dbfft_fd_allgather",
           "dbfft_peer_probe_open", "dbfft_peer_probe_check", "dbfft_peer_probe_close", "dbfft_info", "dbfft_checkpoint",
           "dbfft_restore"]

_lib = None


class DBFFTError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def load_library(path=None):
    """Load libdbfft.so (raises if it was not built: there is no fallback path).
    DBFFT_LIB overrides the path (used to A/B kernel variants built by build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("DBFFT_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_1905_12725_b200.build` (CUDA extension required)")
    lib = ctypes.CDLL(path)
    P, I32, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
    lib.dbfft_create.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double), I32,
                                 ctypes.POINTER(Env), ctypes.POINTER(P)]
    lib.dbfft_destroy.argtypes = [P]
    lib.dbfft_fd_allgather.argtypes = [ctypes.c_char_p, I32, I32, ctypes.POINTER(ctypes.c_int32), I32,
                                       ctypes.POINTER(ctypes.c_int32), I32]
    lib.dbfft_peer_probe_open.argtypes = [ctypes.c_char_p, I32, I32, I32, ctypes.POINTER(ctypes.c_void_p)]
    lib.dbfft_peer_probe_check.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.dbfft_peer_probe_close.argtypes = [P]
    lib.dbfft_last_error.argtypes = [P]
    lib.dbfft_last_error.restype = ctypes.c_char_p
    lib.dbfft_spectral_layout.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.dbfft_set_phases.argtypes = [P, P, I32, I32, ctypes.POINTER(Material)]
    lib.dbfft_apply_K.argtypes = [P, P, P]
    lib.dbfft_apply_K_aug.argtypes = [P, ctypes.POINTER(ctypes.c_uint8), P, ctypes.POINTER(D), P, ctypes.POINTER(D)]
    lib.dbfft_precond.argtypes = [P, P, P]
    lib.dbfft_eval_state.argtypes = [P, P, I32, D]
    lib.dbfft_default_opts.restype = Opts
    lib.dbfft_solve_increment.argtypes = [P, ctypes.POINTER(D), ctypes.POINTER(ctypes.c_uint8), D,
                                          ctypes.POINTER(Opts), ctypes.POINTER(Report)]
    lib.dbfft_get_field.argtypes = [P, I32, P, I32]
    lib.dbfft_profile_enable.argtypes = [P, I32]
    lib.dbfft_profile_read.argtypes = [P, I32, ctypes.POINTER(D), ctypes.POINTER(ctypes.c_int64)]
    lib.dbfft_profile_name.argtypes = [I32]
    lib.dbfft_profile_name.restype = ctypes.c_char_p
    lib.dbfft_profile_count.restype = I32
    lib.dbfft_launch_count.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    lib.dbfft_nccl_unique_id.argtypes = [P]
    lib.dbfft_residuals.argtypes = [P, ctypes.POINTER(D), ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(D)]
    lib.dbfft_incompatibility.argtypes = [P, P, I32, ctypes.POINTER(D)]
    lib.dbfft_get_trace.argtypes = [P, ctypes.POINTER(D), I32, ctypes.POINTER(I32)]
    lib.dbfft_info.argtypes = [P, ctypes.c_char_p, I32]
    lib.dbfft_checkpoint.argtypes = [P, P, ctypes.POINTER(ctypes.c_size_t)]
    lib.dbfft_restore.argtypes = [P, P, ctypes.c_size_t]
    for fn in EXPORTS:
        getattr(lib, fn).restype = getattr(lib, fn).restype if fn in (
            "dbfft_last_error", "dbfft_default_opts", "dbfft_profile_name", "dbfft_profile_count") else ctypes.c_int
    _lib = lib
    return lib


def material_record(m):
    """synth.configs material dict -> dbfft_material (parameters copied, no arithmetic)."""
    rec = Material()
    k = m["kind"]
    if k == "iso":
        rec.kind, vals = MAT_ISO, [m["E"], m["nu"]]
    elif k == "cubic":
        rec.kind, vals = MAT_CUBIC, [m["C11"], m["C12"], m["C44"], *np.asarray(m["R"], float).ravel()]
    elif k == "neohooke":
        rec.kind, vals = MAT_NEOHOOKE, [m["mu"], m["kappa"]]
    elif k == "j2":
        rec.kind, vals = MAT_J2, [m["E"], m["nu"], m["sigma_y"], m["n"], m["edot0"]]
    elif k == "svk":
        rec.kind, vals = MAT_SVK, [m["E"], m["nu"]]
    else:
        raise ValueError(k)
    for i, v in enumerate(vals):
        rec.p[i] = float(v)
    return rec


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr())


def nccl_unique_id_broadcast(rank, process_group=None):
    """Rank 0 creates the NCCL unique id through the library; every rank receives it via
    torch.distributed.broadcast_object_list (host-side bootstrap only)."""
    import torch.distributed as dist
    lib = load_library()
    obj = [None]
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        st = lib.dbfft_nccl_unique_id(buf)
        if st != 0:
            raise DBFFTError(st, lib.dbfft_last_error(None).decode())
        obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=0, group=process_group)
    return ctypes.create_string_buffer(obj[0], 128)


class DBFFT:
    """One DBFFT context on one CUDA device (include/dbfft.h)."""

    def __init__(self, n, L=(1.0, 1.0, 1.0), kinematics="small", device=0, stream=None,
                 world=1, rank=0, loopback=False, process_group=None, transport="nccl", allocator="torch",
                 pencil_rows=1):
        """world > 1: slab decomposition (include/dbfft.h "Distribution").  loopback=True keeps
        all `world` virtual ranks in this process; otherwise NCCL, with the unique id broadcast
        over `process_group` (torch.distributed, any backend).  transport: "nccl" (all-to-all
        exchanges) or "peer" (passes store into the peers' receive buffers, dbfft_env.transport).
        allocator: "torch" (the ctx's device memory from torch's caching allocator, dbfft_env
        dev_alloc / dev_free), "cuda" (cudaMalloc) or a tuple (alloc(nbytes) -> ptr, free(ptr)).
        pencil_rows = Py > 1: 2-D pencil decomposition on a Py x (world / Py) rank grid
        (dbfft_env.pencil_rows), else z-slabs."""
        import torch
        self.torch = torch
        self.lib = load_library()
        self.n = tuple(int(v) for v in n)
        self.kin = 6 if kinematics in ("small", 6) else 9
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.world, self.rank, self.loopback = int(world), int(rank), bool(loopback)
        self.py = max(1, int(pencil_rows))
        self.pz = self.world // self.py
        self._nccl_id = None
        if self.world > 1 and not self.loopback:
            self._nccl_id = nccl_unique_id_broadcast(self.rank, process_group)
        if isinstance(allocator, tuple):  # (alloc(nbytes) -> device pointer, free(ptr)) Python callables
            fa, ff = allocator
            self._alloc = (ALLOC_FN(lambda nbytes, _u: fa(int(nbytes))), FREE_FN(lambda ptr, _u: ff(ptr)))
        elif allocator == "torch":
            self._alloc = torch_allocator(device)   # kept alive as long as the ctx
        elif allocator == "cuda":
            self._alloc = (ALLOC_FN(), FREE_FN())
        else:
            raise ValueError(allocator)
        env = Env(self.rank, self.world, ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id else None,
                  ctypes.c_void_p(self.stream.cuda_stream), device, int(self.loopback), TRANSPORTS[transport],
                  self._alloc[0], self._alloc[1], None, self.py)
        h = ctypes.c_void_p()
        st = self.lib.dbfft_create((ctypes.c_int32 * 3)(*self.n), (ctypes.c_double * 3)(*L), self.kin,
                                   ctypes.byref(env), ctypes.byref(h))
        if st != 0:
            raise DBFFTError(st, self.lib.dbfft_last_error(None).decode())
        self.h = h
        shape = (ctypes.c_int64 * 4)()
        strides = (ctypes.c_int64 * 4)()
        self._check(self.lib.dbfft_spectral_layout(self.h, shape, strides))
        self.spec_shape = tuple(shape)

    def _check(self, st):
        if st != 0:
            raise DBFFTError(st, self.lib.dbfft_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.dbfft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ setup
    def _nloc(self):
        n1, n2, n3 = self.n
        if self.world > 1 and not self.loopback:
            n3 //= self.pz  # NCCL mode: this rank's block [n3/Pz][n2/Py][n1] (z-slabs: Py = 1)
            n2 //= self.py
        return n1 * n2 * n3

    def set_phases(self, phase, materials):
        """phase: integer ids [z][y][x] (numpy array or torch tensor; any integer dtype with values in
        [0, 65535]), host or on this context's device.  The C ABI takes uint16 (include/dbfft.h)."""
        recs = (Material * len(materials))(*[material_record(m) for m in materials])
        torch = self.torch
        if isinstance(phase, torch.Tensor) and phase.device.type != "cuda":
            phase = phase.numpy()
        if isinstance(phase, torch.Tensor):
            if phase.device != self.device:
                raise ValueError(f"set_phases: phase tensor on {phase.device}, context on {self.device}")
            if phase.numel() != self._nloc():
                raise ValueError(f"set_phases: {phase.numel()} ids for {self._nloc()} voxels")
            if phase.dtype in (torch.int16, getattr(torch, "uint16", torch.int16)):
                ph = phase.contiguous()
            else:
                if phase.is_floating_point() or phase.is_complex() or phase.dtype == torch.bool:
                    raise TypeError(f"set_phases: integer phase ids required, got {phase.dtype}")
                t32 = phase.to(torch.int32)
                if int(t32.min()) < 0 or int(t32.max()) > 65535:
                    raise ValueError("set_phases: phase ids outside [0, 65535]")
                ph = torch.where(t32 >= 32768, t32 - 65536, t32).to(torch.int16).contiguous()  # uint16 bits
            self._check(self.lib.dbfft_set_phases(self.h, _dptr(ph), 1, len(materials), recs))
            return
        arr = np.asarray(phase)
        if arr.dtype != np.uint16:
            if not np.issubdtype(arr.dtype, np.integer):
                raise TypeError(f"set_phases: integer phase ids required, got {arr.dtype}")
            if arr.size and (arr.min() < 0 or arr.max() > 65535):
                raise ValueError("set_phases: phase ids outside [0, 65535]")
        if arr.size != self._nloc():
            raise ValueError(f"set_phases: {arr.size} ids for {self._nloc()} voxels")
        ph = np.ascontiguousarray(arr, dtype=np.uint16)
        self._check(self.lib.dbfft_set_phases(self.h, ph.ctypes.data_as(ctypes.c_void_p), 0, len(materials), recs))

    def empty_spectral(self):
        return self.torch.empty(self.spec_shape, dtype=self.torch.complex128, device=self.device)

    def _spec_in(self, t, name):
        """A spectral vector argument: complex128, this device, spec_shape; returned contiguous (the
        caller keeps the returned tensor alive until the C call returns)."""
        torch = self.torch
        if not isinstance(t, torch.Tensor) or t.dtype != torch.complex128 or t.device != self.device \
                or tuple(t.shape) != self.spec_shape:
            raise ValueError(f"{name}: complex128 tensor of shape {self.spec_shape} on {self.device} required, got "
                             f"{getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))} on {getattr(t, 'device', '?')}")
        return t.contiguous()

    def _spec_out(self, out, name):
        if out is None:
            return self.empty_spectral()
        o = self._spec_in(out, name)
        if o.data_ptr() != out.data_ptr():
            raise ValueError(f"{name}: output tensor must be contiguous")
        return out

    # ------------------------------------------------------------------ operator
    def apply_K(self, u_hat, out=None):
        u = self._spec_in(u_hat, "apply_K(u_hat)")
        out = self._spec_out(out, "apply_K(out)")
        self._check(self.lib.dbfft_apply_K(self.h, _dptr(u), _dptr(out)))
        return out

    def apply_K_aug(self, mask, u_hat, e, out=None):
        u = self._spec_in(u_hat, "apply_K_aug(u_hat)")
        out = self._spec_out(out, "apply_K_aug(out)")
        m = (ctypes.c_uint8 * 9)(*np.asarray(mask, np.uint8).ravel())
        ein = (ctypes.c_double * 9)(*np.asarray(e, float).ravel())
        rout = (ctypes.c_double * 9)()
        self._check(self.lib.dbfft_apply_K_aug(self.h, m, _dptr(u), ein, _dptr(out), rout))
        return out, np.array(rout[:]).reshape(3, 3)

    def precond(self, r_hat, out=None):
        r = self._spec_in(r_hat, "precond(r_hat)")
        out = self._spec_out(out, "precond(out)")
        self._check(self.lib.dbfft_precond(self.h, _dptr(r), _dptr(out)))
        return out

    def eval_state(self, field, dt=1.0):
        """field: real [3,3,z,y,x] eps (small strain) or F (finite), numpy or a float64 tensor on
        this device."""
        torch = self.torch
        if isinstance(field, torch.Tensor) and field.device.type != "cuda":
            field = field.numpy()
        if isinstance(field, torch.Tensor):
            if field.dtype != torch.float64 or field.device != self.device or field.numel() != 9 * self._nloc():
                raise ValueError(f"eval_state: float64 tensor of {9 * self._nloc()} values on {self.device} required")
            f = field.contiguous()
            self._check(self.lib.dbfft_eval_state(self.h, _dptr(f), 1, float(dt)))
            return
        f = np.ascontiguousarray(field, dtype=np.float64)
        if f.size != 9 * self._nloc():
            raise ValueError(f"eval_state: {f.size} values for a 9 x {self._nloc()} field")
        self._check(self.lib.dbfft_eval_state(self.h, f.ctypes.data_as(ctypes.c_void_p), 0, float(dt)))

    # ------------------------------------------------------------------ solve
    def solve_increment(self, target, mask, dt=1.0, raise_on_error=True, **opts):
        o = self.lib.dbfft_default_opts()
        for k, v in opts.items():
            setattr(o, k, v)
        t = (ctypes.c_double * 9)(*np.asarray(target, float).ravel())
        m = (ctypes.c_uint8 * 9)(*np.asarray(mask, np.uint8).ravel())
        rep = Report()
        st = self.lib.dbfft_solve_increment(self.h, t, m, float(dt), ctypes.byref(o), ctypes.byref(rep))
        out = dict(status=STATUS.get(st, st), converged=bool(rep.converged), cg_iters=rep.cg_iters,
                   newton_iters=rep.newton_iters, eps_eq=rep.eps_eq, eps_load=rep.eps_load,
                   max_dgrad=rep.max_dgrad, macro_strain=np.array(rep.macro_strain[:]).reshape(3, 3),
                   macro_stress=np.array(rep.macro_stress[:]).reshape(3, 3), bad_voxel=rep.bad_voxel,
                   seconds=rep.seconds)
        if st != 0 and raise_on_error:
            raise DBFFTError(st, self.lib.dbfft_last_error(self.h).decode())
        return out

    def get_field(self, which, on_device=False, pinned=False, out=None):
        """Committed field (C ABI dbfft_get_field).  Host results land in a fresh numpy array;
        pinned=True allocates it in page-locked memory (faster D2H copy); `out` (a C-contiguous
        float64 host array of the field's size, e.g. a reused pinned buffer) receives it instead."""
        n1, n2, n3 = self.n
        if self.world > 1 and not self.loopback:
            n3 //= self.pz  # NCCL mode: this rank's block [n3/Pz][n2/Py][n1] (z-slabs: Py = 1)
            n2 //= self.py
        N = n1 * n2 * n3
        if out is not None:
            ncomp = {FIELD_U: 3, FIELD_TANGENT: 81}.get(which, 9)
            if which == FIELD_U_HAT or not isinstance(out, np.ndarray) or out.dtype != np.float64 \
                    or out.size != ncomp * N or not out.flags["C_CONTIGUOUS"]:
                raise ValueError("get_field(out=): a C-contiguous float64 host array of the field's size")
            self._check(self.lib.dbfft_get_field(self.h, which, out.ctypes.data_as(ctypes.c_void_p), 0))
            return out
        if which == FIELD_U_HAT:
            out = self.empty_spectral()
            self._check(self.lib.dbfft_get_field(self.h, which, _dptr(out), 1))
            return out
        ncomp = {FIELD_U: 3, FIELD_TANGENT: 81}.get(which, 9)
        if on_device:
            out = self.torch.empty((ncomp, n3, n2, n1), dtype=self.torch.float64, device=self.device)
            self._check(self.lib.dbfft_get_field(self.h, which, _dptr(out), 1))
            return out
        if pinned:
            out = self.torch.empty((ncomp, n3, n2, n1), dtype=self.torch.float64, pin_memory=True).numpy()
        else:
            out = np.empty((ncomp, n3, n2, n1))
        self._check(self.lib.dbfft_get_field(self.h, which, out.ctypes.data_as(ctypes.c_void_p), 0))
        if ncomp == 9:
            out = out.reshape(3, 3, n3, n2, n1)
        elif ncomp == 81:
            out = out.reshape(3, 3, 3, 3, n3, n2, n1)
        return out

    # ------------------------------------------------------------------ residual monitors
    def residuals(self, target, mask):
        """(equilibrium, compatibility, loading) of the committed state."""
        t = (ctypes.c_double * 9)(*np.asarray(target, float).ravel())
        m = (ctypes.c_uint8 * 9)(*np.asarray(mask, np.uint8).ravel())
        out = (ctypes.c_double * 3)()
        self._check(self.lib.dbfft_residuals(self.h, t, m, out))
        return dict(equilibrium=out[0], compatibility=out[1], loading=out[2])

    def trace(self):
        """(eps_eq, eps_load) per PCG iteration of the last solve_increment, shape (n, 2)."""
        n = ctypes.c_int32()
        self._check(self.lib.dbfft_get_trace(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(n.value, 1), 2))
        self._check(self.lib.dbfft_get_trace(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n.value,
                                             ctypes.byref(n)))
        return out[:n.value]

    def incompatibility(self, field):
        """max|curl curl eps| (small) or max|curl F| (finite) of a real [3,3,z,y,x] field."""
        f = np.ascontiguousarray(np.asarray(field, np.float64).reshape(9, -1))
        out = ctypes.c_double()
        self._check(self.lib.dbfft_incompatibility(self.h, f.ctypes.data_as(ctypes.c_void_p), 0, ctypes.byref(out)))
        return out.value

    # ------------------------------------------------------------------ checkpoint / resume
    def checkpoint(self):
        """The committed state as bytes (dbfft_checkpoint)."""
        n = ctypes.c_size_t(0)
        self._check(self.lib.dbfft_checkpoint(self.h, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self._check(self.lib.dbfft_checkpoint(self.h, buf, ctypes.byref(n)))
        return buf.raw[: n.value]

    def restore(self, blob):
        """Install a checkpoint (after set_phases with the same microstructure)."""
        buf = ctypes.create_string_buffer(bytes(blob), len(blob))
        self._check(self.lib.dbfft_restore(self.h, buf, len(blob)))

    # ------------------------------------------------------------------ profiling
    def info(self):
        """dbfft_info: device, ranks, transport, NCCL communicator, how the last PCG loop ran."""
        import json
        buf = ctypes.create_string_buffer(1024)
        self._check(self.lib.dbfft_info(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def profile(self, enable=True):
        self._check(self.lib.dbfft_profile_enable(self.h, int(enable)))

    def launch_count(self):
        n = ctypes.c_int64()
        self._check(self.lib.dbfft_launch_count(self.h, ctypes.byref(n)))
        return n.value

    def profile_read(self):
        res = {}
        for k in range(self.lib.dbfft_profile_count()):
            ms = ctypes.c_double()
            n = ctypes.c_int64()
            self._check(self.lib.dbfft_profile_read(self.h, k, ctypes.byref(ms), ctypes.byref(n)))
            res[self.lib.dbfft_profile_name(k).decode()] = (ms.value, n.value)
        return res
