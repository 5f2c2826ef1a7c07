"""B200-native synchronous lazy-PCA sweep (arXiv 2507.14869) -- thin Python binding.

Every entry point has the same name as the C ABI in ``include/pca.h`` and only
marshals arguments: all device work runs in ``libpca_b200.so`` (hand-written sm_100a
CUDA).  PyTorch is used for device memory (the workspace and image tensors) and streams.
There is no CPU fallback: if the extension is missing or no CUDA device is present,
``lib()`` / ``PcaContext`` raise.

Image arguments are uint8 tensors (or NumPy arrays for host data) shaped
``[batch, rows, width]`` (a 2-D ``[rows, width]`` is accepted for batch == 1).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCA_B200_LIB_OVERRIDE") or os.path.join(_PKG, "libpca_b200.so")

PCA_OK, PCA_EINVAL, PCA_ESTATE, PCA_ECUDA, PCA_ENCCL, PCA_ENOSPACE, PCA_EUNSUPPORTED = (
    0, -1, -2, -3, -4, -5, -6)
EST_LAST, EST_MPM, EST_MARGINALS, EST_CM = 0, 1, 2, 3
KERNEL_AUTO, KERNEL_GENERAL, KERNEL_BINARY, KERNEL_TABLE, KERNEL_PACKED = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "PCA_OK", -1: "PCA_EINVAL", -2: "PCA_ESTATE", -3: "PCA_ECUDA",
                -4: "PCA_ENCCL", -5: "PCA_ENOSPACE", -6: "PCA_EUNSUPPORTED"}

# every symbol include/pca.h declares
EXPORTS = ["pca_abi_version", "pca_workspace_bytes", "pca_init", "pca_reset", "pca_sweep",
           "pca_gibbs_sweep", "pca_estimate", "pca_metric_sums", "pca_psnr_ssim", "pca_finalize",
           "pca_stage_truth", "pca_changed_sites",
           "pca_ssim_windowed", "pca_read_state",
           "pca_write_state", "pca_read_counts", "pca_write_counts", "pca_set_step",
           "pca_get_stats", "pca_halo_ptrs", "pca_nccl_unique_id", "pca_attach_nccl", "pca_sync",
           "pca_destroy", "pca_last_error", "pca_peer_info", "pca_ipc_handle", "pca_open_peer",
           "pca_close_peer", "pca_attach_peers", "pca_stage_input", "pca_reset_staged",
           "pca_finalize_async"]


class PcaError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class pca_config(ctypes.Structure):
    """Mirror of ``pca_config`` (include/pca.h)."""

    _fields_ = [
        ("height", ctypes.c_int32), ("width", ctypes.c_int32), ("batch", ctypes.c_int32),
        ("levels", ctypes.c_int32), ("neighborhood", ctypes.c_int32),
        ("periodic", ctypes.c_int32), ("J", ctypes.c_double), ("q", ctypes.c_double),
        ("sigma", ctypes.c_double), ("beta0", ctypes.c_double), ("beta_step", ctypes.c_double),
        ("beta_period", ctypes.c_int32), ("chain0", ctypes.c_int32),
        ("coef_scale", ctypes.c_double), ("seed", ctypes.c_uint64),
        ("mpm_burn_in", ctypes.c_int32), ("row0", ctypes.c_int32), ("rows", ctypes.c_int32),
        ("kernel", ctypes.c_int32), ("rows_per_thread", ctypes.c_int32),
        ("sweeps_per_pass", ctypes.c_int32), ("inertia_p", ctypes.c_int32),
        ("packed_io", ctypes.c_int32), ("graphs", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3),
    ]


class pca_stats(ctypes.Structure):
    _fields_ = [("sweeps_done", ctypes.c_int64), ("counted_sweeps", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("sweep_launches", ctypes.c_int64),
                ("beta", ctypes.c_double), ("kernel", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("graph_replays", ctypes.c_int64)]


class pca_peer(ctypes.Structure):
    """A neighbouring rank's buffers and phase words (device-initiated halo exchange)."""
    _fields_ = [("x", ctypes.c_void_p * 2), ("flags", ctypes.c_void_p), ("ipc_base", ctypes.c_void_p),
                ("rows", ctypes.c_int32), ("batch", ctypes.c_int32), ("chain_stride", ctypes.c_int64)]


class pca_halo(ctypes.Structure):
    _fields_ = [("send_top", ctypes.c_void_p), ("send_bottom", ctypes.c_void_p),
                ("recv_top", ctypes.c_void_p), ("recv_bottom", ctypes.c_void_p),
                ("row_bytes", ctypes.c_size_t), ("chain_stride", ctypes.c_size_t),
                ("g_send_top", ctypes.c_void_p), ("g_send_bottom", ctypes.c_void_p),
                ("g_recv_top", ctypes.c_void_p), ("g_recv_bottom", ctypes.c_void_p),
                ("g_row_bytes", ctypes.c_size_t), ("g_chain_stride", ctypes.c_size_t)]


_lib = None


def lib():
    """Load libpca_b200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run paper_2507_14869_b200.build.build() "
                               "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        cfgp = ctypes.POINTER(pca_config)
        sigs = {
            "pca_abi_version": (i32, []),
            "pca_workspace_bytes": (sz, [cfgp]),
            "pca_init": (i32, [ctypes.POINTER(vp), cfgp, vp, sz, vp, vp, vp]),
            "pca_reset": (i32, [vp, vp, vp]),
            "pca_sweep": (i32, [vp, i32]),
            "pca_gibbs_sweep": (i32, [vp, i32]),
            "pca_estimate": (i32, [vp, i32, vp]),
            "pca_metric_sums": (i32, [vp, vp, i32, vp]),
            "pca_psnr_ssim": (i32, [vp, vp, i32, vp, vp]),
            "pca_ssim_windowed": (i32, [vp, vp, i32, vp]),
            "pca_finalize": (i32, [vp, vp, vp, vp, vp]),
            "pca_finalize_async": (i32, [vp, vp, vp, vp, vp]),
            "pca_stage_truth": (i32, [vp, vp]),
            "pca_changed_sites": (i32, [vp, vp]),
            "pca_read_state": (i32, [vp, vp]),
            "pca_write_state": (i32, [vp, vp]),
            "pca_read_counts": (i32, [vp, vp]),
            "pca_write_counts": (i32, [vp, vp, i64]),
            "pca_set_step": (i32, [vp, i64]),
            "pca_get_stats": (i32, [vp, ctypes.POINTER(pca_stats)]),
            "pca_halo_ptrs": (i32, [vp, ctypes.POINTER(pca_halo)]),
            "pca_peer_info": (i32, [vp, ctypes.POINTER(pca_peer)]),
            "pca_stage_input": (i32, [vp, vp]),
            "pca_reset_staged": (i32, [vp]),
            "pca_ipc_handle": (i32, [vp, vp, ctypes.POINTER(ctypes.c_uint64)]),
            "pca_open_peer": (i32, [vp, vp, ctypes.c_uint64, ctypes.POINTER(pca_config), ctypes.POINTER(pca_peer)]),
            "pca_close_peer": (i32, [ctypes.POINTER(pca_peer)]),
            "pca_attach_peers": (i32, [vp, ctypes.POINTER(pca_peer), ctypes.POINTER(pca_peer)]),
            "pca_nccl_unique_id": (i32, [vp]),
            "pca_attach_nccl": (i32, [vp, vp, i32, i32]),
            "pca_sync": (i32, [vp]),
            "pca_destroy": (i32, [vp]),
            "pca_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != PCA_OK:
        raise PcaError(status, where, lib().pca_last_error().decode())


def make_config(height, width, levels, *, batch=1, neighborhood=8, periodic=False, J=1.0 / 3.0,
                q=0.51, sigma=0.25, beta0=1.25, beta_step=0.25, beta_period=250, chain0=0,
                coef_scale=1.0, seed=0, mpm_burn_in=-1, row0=0, rows=0, kernel=KERNEL_AUTO,
                rows_per_thread=0, sweeps_per_pass=0, inertia_p=0, packed_io=0, graphs=0) -> pca_config:
    """pca_config with the paper's defaults (J = 1/3, q = 0.51, beta
    1.25 + 0.25 every 250 sweeps; Moore-8 neighbourhood, free boundary)."""
    c = pca_config()
    c.height, c.width, c.batch, c.levels = int(height), int(width), int(batch), int(levels)
    c.neighborhood, c.periodic = int(neighborhood), int(bool(periodic))
    c.J, c.q, c.sigma = float(J), float(q), float(sigma)
    c.beta0, c.beta_step, c.beta_period = float(beta0), float(beta_step), int(beta_period)
    c.chain0, c.coef_scale, c.seed = int(chain0), float(coef_scale), int(seed) & (2**64 - 1)
    c.mpm_burn_in, c.row0, c.rows = int(mpm_burn_in), int(row0), int(rows)
    c.kernel, c.rows_per_thread = int(kernel), int(rows_per_thread)
    c.sweeps_per_pass = int(sweeps_per_pass)
    c.inertia_p = int(inertia_p)
    c.packed_io = int(packed_io)
    c.graphs = int(graphs)
    return c


def pca_workspace_bytes(cfg: pca_config) -> int:
    n = lib().pca_workspace_bytes(ctypes.byref(cfg))
    if n == 0:
        raise PcaError(PCA_EINVAL, "pca_workspace_bytes", lib().pca_last_error().decode())
    return int(n)


def pca_close_peer(peer: pca_peer):
    _check(lib().pca_close_peer(ctypes.byref(peer)), "pca_close_peer")


def pca_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().pca_nccl_unique_id(buf), "pca_nccl_unique_id")
    return buf.raw


def pack_bits(img) -> np.ndarray:
    """Dense 0/1 labels [..., W] -> the packed_io layout [..., ceil(W/8)] (LSB = first column)."""
    return np.packbits(np.asarray(img, np.uint8) & 1, axis=-1, bitorder="little")


def unpack_bits(bits, width: int) -> np.ndarray:
    """The packed_io layout -> dense 0/1 labels [..., width]."""
    return np.unpackbits(np.asarray(bits, np.uint8), axis=-1, count=width, bitorder="little")


def _ptr(a) -> int:
    """Address of a torch tensor (device or host) or a NumPy array (host)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    assert a.is_contiguous(), "tensor must be contiguous"
    return a.data_ptr()


class PcaContext:
    """One pca_ctx: a lattice (or row strip) x batch of chains on the current CUDA device.

    The workspace is a torch uint8 CUDA tensor owned by this object.  ``stream`` defaults
    to torch's current stream."""

    def __init__(self, cfg: pca_config, g, x0=None, stream=None, device=None, guard: int = 0):
        """guard > 0 (testing): that many bytes after the workspace are filled with 0xA5;
        guard_intact() tells whether any call wrote past the workspace's end."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("PcaContext needs a CUDA device (no CPU fallback)")
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.rows = cfg.rows if cfg.rows else cfg.height
        self.shape = (cfg.batch, self.rows, cfg.width)
        # image arguments / results: dense uint8, or bit-packed rows when cfg.packed_io
        self.image_shape = (cfg.batch, self.rows, (cfg.width + 7) // 8) if cfg.packed_io else self.shape
        nbytes = pca_workspace_bytes(cfg)
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(nbytes + 256 + guard, dtype=torch.uint8, device=self.device)
            off = (-self.workspace.data_ptr()) % 256
            self._ws_ptr = self.workspace.data_ptr() + off
            self._guard = self.workspace[off + nbytes:off + nbytes + guard] if guard else None
            if guard:
                self._guard.fill_(0xA5)
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            self._keep = [g, x0]
            h = ctypes.c_void_p()
            _check(lib().pca_init(ctypes.byref(h), ctypes.byref(cfg), self._ws_ptr, nbytes,
                                  _ptr(g), _ptr(x0), self.stream.cuda_stream), "pca_init")
        self.handle = h
        self._keep = None
        # host buffers a copy-stream transfer may still read or write: staged
        # inputs (pca_stage_input) and asynchronous MPM images (pca_finalize_async).  They are
        # released only once a call has provably waited for the copy on the host, never at the
        # return of the call that enqueued or consumed it.
        self._staged_inputs = []   # [buffer, consumed by a reset_staged?]
        self._async_outputs = []

    def _synced_main(self):
        """The library host-synchronised the main stream after waiting on the copy events:
        inputs already consumed by a staged reset, and earlier asynchronous images (every
        synchronising call waits for the previous image copy first), are complete."""
        self._staged_inputs = [e for e in self._staged_inputs if not e[1]]
        self._async_outputs = []

    # ---- ABI wrappers (same names) ----
    def pca_reset(self, g=None, x0=None):
        _check(lib().pca_reset(self.handle, _ptr(g), _ptr(x0)), "pca_reset")

    def pca_stage_input(self, g):
        """Copy the next reset's g on the internal copy stream (overlaps the work after it)."""
        self._staged_inputs.append([g, False])  # alive until a host sync covers the copy
        _check(lib().pca_stage_input(self.handle, _ptr(g)), "pca_stage_input")

    def pca_reset_staged(self):
        _check(lib().pca_reset_staged(self.handle), "pca_reset_staged")
        for e in self._staged_inputs:  # the main stream now waits for these copies
            e[1] = True

    def pca_sweep(self, n: int):
        _check(lib().pca_sweep(self.handle, int(n)), "pca_sweep")

    def pca_gibbs_sweep(self, n: int):
        _check(lib().pca_gibbs_sweep(self.handle, int(n)), "pca_gibbs_sweep")

    def pca_estimate(self, kind: int, out):
        _check(lib().pca_estimate(self.handle, int(kind), _ptr(out)), "pca_estimate")
        self._synced_main()
        return out

    def pca_metric_sums(self, truth, kind: int) -> np.ndarray:
        s = np.zeros((self.cfg.batch, 8), np.int64)
        _check(lib().pca_metric_sums(self.handle, _ptr(truth), int(kind), s.ctypes.data),
               "pca_metric_sums")
        return s

    def pca_psnr_ssim(self, truth, kind: int):
        p = np.zeros(self.cfg.batch, np.float64)
        s = np.zeros(self.cfg.batch, np.float64)
        _check(lib().pca_psnr_ssim(self.handle, _ptr(truth), int(kind), p.ctypes.data,
                                   s.ctypes.data), "pca_psnr_ssim")
        self._synced_main()
        return p, s

    def pca_stage_truth(self, truth):
        """Copy the truth on the context's copy stream (overlaps later sweeps); the host buffer
        must stay alive until the next pca_finalize(None, ...) returns."""
        self._staged_truth = truth  # keep the host buffer alive
        _check(lib().pca_stage_truth(self.handle, _ptr(truth)), "pca_stage_truth")

    def pca_finalize(self, truth, mpm_out=None):
        """MPM image (into mpm_out when given) and PSNR / SSIM of LAST and MPM in one pass:
        returns (psnr, ssim), each [batch][2] (column 0 LAST, column 1 MPM).  truth None:
        the image staged with pca_stage_truth."""
        p = np.zeros((self.cfg.batch, 2), np.float64)
        s = np.zeros((self.cfg.batch, 2), np.float64)
        _check(lib().pca_finalize(self.handle, _ptr(truth), _ptr(mpm_out), p.ctypes.data,
                                  s.ctypes.data), "pca_finalize")
        self._synced_main()
        return p, s

    def pca_finalize_async(self, truth, mpm_out):
        """pca_finalize with the MPM image's copy into host mpm_out on the copy stream: the
        image may still be in flight at return (pca_sync waits for it); keep mpm_out alive
        and unread until then."""
        p = np.zeros((self.cfg.batch, 2), np.float64)
        s = np.zeros((self.cfg.batch, 2), np.float64)
        # the previous image stays referenced until this call has waited for its copy
        self._async_outputs.append(mpm_out)
        _check(lib().pca_finalize_async(self.handle, _ptr(truth), _ptr(mpm_out), p.ctypes.data,
                                        s.ctypes.data), "pca_finalize_async")
        self._synced_main()
        self._async_outputs = [mpm_out]  # in flight until the next synchronising call
        return p, s

    def pca_ssim_windowed(self, truth, kind: int):
        s = np.zeros(self.cfg.batch, np.float64)
        _check(lib().pca_ssim_windowed(self.handle, _ptr(truth), int(kind), s.ctypes.data),
               "pca_ssim_windowed")
        return s

    def pca_read_state(self, out):
        _check(lib().pca_read_state(self.handle, _ptr(out)), "pca_read_state")
        return out

    def pca_write_state(self, x):
        _check(lib().pca_write_state(self.handle, _ptr(x)), "pca_write_state")

    def pca_read_counts(self, out):
        _check(lib().pca_read_counts(self.handle, _ptr(out)), "pca_read_counts")
        return out

    def pca_write_counts(self, c, counted: int):
        _check(lib().pca_write_counts(self.handle, _ptr(c), int(counted)), "pca_write_counts")

    def pca_set_step(self, t: int):
        _check(lib().pca_set_step(self.handle, int(t)), "pca_set_step")

    def pca_changed_sites(self) -> np.ndarray:
        """Sites whose label changed in the most recent sweep, per chain."""
        out = np.zeros(self.cfg.batch, np.int64)
        _check(lib().pca_changed_sites(self.handle, out.ctypes.data), "pca_changed_sites")
        return out

    def pca_get_stats(self) -> pca_stats:
        st = pca_stats()
        _check(lib().pca_get_stats(self.handle, ctypes.byref(st)), "pca_get_stats")
        return st

    def pca_halo_ptrs(self) -> pca_halo:
        h = pca_halo()
        _check(lib().pca_halo_ptrs(self.handle, ctypes.byref(h)), "pca_halo_ptrs")
        return h

    def pca_peer_info(self) -> pca_peer:
        q = pca_peer()
        _check(lib().pca_peer_info(self.handle, ctypes.byref(q)), "pca_peer_info")
        return q

    def pca_ipc_handle(self) -> tuple[bytes, int]:
        """(64-byte CUDA IPC handle of the workspace's allocation, workspace offset in it)."""
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64()
        _check(lib().pca_ipc_handle(self.handle, buf, ctypes.byref(off)), "pca_ipc_handle")
        return buf.raw, int(off.value)

    def pca_open_peer(self, handle: bytes, offset: int, peer_cfg: pca_config) -> pca_peer:
        """Map another process's workspace (its pca_ipc_handle) into this context's device."""
        q = pca_peer()
        buf = ctypes.create_string_buffer(handle, 64)
        _check(lib().pca_open_peer(self.handle, buf, int(offset), ctypes.byref(peer_cfg), ctypes.byref(q)),
               "pca_open_peer")
        return q

    def pca_attach_peers(self, up: pca_peer | None, down: pca_peer | None):
        """Device-initiated halo exchange with the ranks above (up) / below (down) this strip."""
        _check(lib().pca_attach_peers(self.handle, ctypes.byref(up) if up is not None else None,
                                      ctypes.byref(down) if down is not None else None), "pca_attach_peers")

    def pca_attach_nccl(self, uid: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(uid, 128)
        _check(lib().pca_attach_nccl(self.handle, buf, int(nranks), int(rank)), "pca_attach_nccl")

    def pca_sync(self):
        _check(lib().pca_sync(self.handle), "pca_sync")
        self._staged_inputs = []
        self._async_outputs = []

    def pca_destroy(self):
        if getattr(self, "handle", None):
            lib().pca_destroy(self.handle)  # waits for every stream, copies included
            self.handle = None
            self._staged_inputs = []
            self._async_outputs = []

    def guard_intact(self) -> bool:
        """No byte after the workspace's end was written (contexts made with guard > 0)."""
        import torch

        torch.cuda.synchronize(self.device)
        return bool((self._guard == 0xA5).all().item())

    # ---- conveniences (host NumPy results) ----
    def state(self) -> np.ndarray:
        return self.pca_read_state(np.empty(self.image_shape, np.uint8))

    def counts(self) -> np.ndarray:
        planes = 1 if self.cfg.levels == 2 else self.cfg.levels
        shape = (self.cfg.batch, self.rows, self.cfg.width) if planes == 1 else \
            (self.cfg.batch, planes, self.rows, self.cfg.width)
        return self.pca_read_counts(np.empty(shape, np.uint16))

    def estimate(self, kind: int) -> np.ndarray:
        if kind in (EST_LAST, EST_MPM):
            out = np.empty(self.image_shape, np.uint8)
        elif kind == EST_CM:
            out = np.empty(self.shape, np.float32)
        else:
            out = np.empty((self.cfg.batch, self.cfg.levels, self.rows, self.cfg.width), np.float32)
        return self.pca_estimate(kind, out)

    def __del__(self):
        try:
            self.pca_destroy()
        except Exception:
            pass
