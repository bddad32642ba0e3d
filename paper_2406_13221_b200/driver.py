"""Fused training driver: the reference's ``train_encrypted`` loop
(enctrain.py:303-449) with each iteration issued as one native call
(``helr_nag_iteration``) over a whole batch of row blocks, optionally
replayed from a captured CUDA graph.

Host responsibilities (this module):
- ``plan_iteration``: exact-scale bookkeeping for the depth-7 schedule and
  the per-limb integer constants it needs.  All scales are
  fp64 and tracked exactly; every constant product encodes its constant at
  the scale that makes the product land on a chosen target, so additions
  always see equal scales.
- ``FusedTrainer``: client preparation (pack + encrypt Z and B̄ on the
  device), keys, the refresh policy (same arithmetic as
  ``bootstrap_policy``, enctrain.py:242-255), decryption of the weights.

Device responsibilities: everything between the weights going in and the
updated weights coming out (csrc/nag.cu).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .ckks import GpuContext
from .encoding import BlockLayout, pack_matrix_array, plan_layout, replicate_rows
from .optimizer import ALPHA0_INIT, BASELINE_CUBIC, PolyApprox, lr_at, merge_bbar, next_alpha, scaler_for
from .shard import partition

__all__ = ["IterPlan", "plan_iteration", "NagArgs", "FusedTrainer", "NCONST", "ITER_DEPTH"]

NCONST = 10
ITER_DEPTH = 7  # rescales per iteration


def rotsum_groups(log_total: int, max_bits: int) -> list:
    """Bit-widths of the hoisted groups of a grouped rotate-and-sum over
    2^log_total rotations (same rule as helr_rotsum_groups, csrc/nag.cu)."""
    if log_total <= 0 or max_bits <= 0:
        return []
    ng = -(-log_total // max_bits)
    base, rem = divmod(log_total, ng)
    return [base + 1 if j < rem else base for j in range(ng)]


def grouped_steps(log_total: int, max_bits: int, stride: int = 1) -> list:
    """Rotation steps per group (key order of helr_nag_args.rot_*)."""
    out, off = [], 0
    for bits in rotsum_groups(log_total, max_bits):
        out.append([(stride * k) << off for k in range(1, 1 << bits)])
        off += bits
    return out


class NagArgs(ctypes.Structure):
    """Mirror of ``helr_nag_args`` (include/helr_ckks.h)."""

    _fields_ = [
        ("z", ctypes.c_void_p), ("rows", ctypes.c_int), ("cols", ctypes.c_int),
        ("log_g", ctypes.c_int), ("log_m", ctypes.c_int),
        ("w", ctypes.c_void_p), ("v", ctypes.c_void_p), ("bbar", ctypes.c_void_p), ("lw", ctypes.c_int),
        ("rlk", ctypes.c_void_p),
        ("rot_left", ctypes.POINTER(ctypes.c_void_p)), ("rot_right", ctypes.POINTER(ctypes.c_void_p)),
        ("rot_rows", ctypes.POINTER(ctypes.c_void_p)),
        ("mask_pt", ctypes.c_void_p), ("consts", ctypes.c_void_p), ("grad", ctypes.c_void_p),
        ("phase", ctypes.c_int), ("log_baby", ctypes.c_int), ("log_baby_rows", ctypes.c_int),
    ]


def _bind(lib):
    if getattr(lib, "_nag_bound", False):
        return
    lib.helr_nag_iteration.argtypes = [ctypes.c_void_p, ctypes.POINTER(NagArgs), ctypes.c_void_p]
    lib.helr_nag_iteration.restype = ctypes.c_int
    lib.helr_nag_graph_capture.argtypes = [ctypes.c_void_p, ctypes.POINTER(NagArgs), ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_void_p)]
    lib.helr_nag_graph_capture.restype = ctypes.c_int
    lib.helr_nag_graph_update.argtypes = [ctypes.c_void_p, ctypes.POINTER(NagArgs), ctypes.c_void_p, ctypes.c_void_p]
    lib.helr_nag_graph_update.restype = ctypes.c_int
    lib.helr_nag_graph_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.helr_nag_graph_launch.restype = ctypes.c_int
    lib.helr_nag_graph_destroy.argtypes = [ctypes.c_void_p]
    lib.helr_nag_graph_destroy.restype = ctypes.c_int
    lib._nag_bound = True


# ---------------------------------------------------------------- planning
@dataclass
class IterPlan:
    lw: int
    consts: np.ndarray          # uint64 [NCONST][L]
    ints: list                  # the signed integer constants (host-side record)
    mask_scale: float
    s_out: float
    scales: dict = field(default_factory=dict)


def _rint(x: float) -> int:
    return int(np.rint(x))


OUT_SCALE_BITS = 50  # scale of W', V' at the bottom level: |W| < q_0 / 2^51 = 2^9
BBAR_EXTRA_BITS = 6  # B̄ encrypted up to 2^6 above s_top / max|B̄| (see FusedTrainer._prepare)


def plan_iteration(ck, lw: int, s_w: float, s_v: float, s_z: float, s_b: float, qpoly, mult: float,
                   eta: float, out_bits: int = OUT_SCALE_BITS) -> IterPlan:
    """Constants of one depth-7 iteration starting with W, V at level ``lw``.

    qpoly = (q0, q1, q2, q3): coefficients of 1 - sigmoid_poly (the
    complement, enctrain.py:155-159, sigmoid.py:72-76); mult = 1 + gamma
    (enhanced) or gamma (baseline), eta = (1 - alpha0) / alpha1
    (enctrain.py:362-366, 224-229).

    Precision: every integer constant is kept >= 2^30 (relative rounding
    <= 2^-30): the NAG constants scale with s_out / s_d, so W', V' land on
    2^out_bits rather than the canonical bottom-level scale, and B̄ arrives
    pre-scaled (s_b = 2^(40 + k) / max|B̄|, k <= 6) so its encryption noise
    is negligible.
    """
    if lw < ITER_DEPTH or lw >= ck.L:
        raise ValueError(f"iteration needs W at a level in [{ITER_DEPTH}, {ck.L}), got {lw}")
    q = [float(x) for x in ck.q]
    D = ck.level_scales
    l = lw
    q0, q1, q2, q3 = qpoly
    s_p = s_z * s_w / q[l]
    s_u = D[l - 2]
    mask_scale = s_u * q[l - 1] / s_p
    s_u2 = s_u * s_u / q[l - 2]
    s_s = D[l - 5]
    s_c = s_s * q[l - 4] / s_z
    s_t = s_c * q[l - 3] / s_u2
    c3 = _rint(q3 * s_t * q[l - 2] / s_u)
    c1 = _rint(q1 * s_c * q[l - 3] / s_u)
    c2 = _rint(q2 * s_c * q[l - 3] / s_u2)
    c0 = _rint(q0 * s_c)
    s_d = s_s * s_b / q[l - 5]
    s_out = float(2 ** out_bits) if l - 7 == 0 else D[l - 7]
    f = s_out * q[l - 6]
    cw1 = _rint(f / s_w)
    ca1 = _rint(mult * f / s_d)
    cw2 = _rint((1.0 - eta) * f / s_w)
    cv2 = _rint(eta * f / s_v)
    ca2 = _rint((1.0 - eta) * mult * f / s_d)
    ints = [c3, c1, c2, c0, cw1, ca1, cw2, cv2, ca2, 0]
    consts = np.zeros((NCONST, ck.L), dtype=np.uint64)
    for k, v in enumerate(ints):
        consts[k] = [v % p for p in ck.q]
    return IterPlan(lw=lw, consts=consts, ints=ints, mask_scale=mask_scale, s_out=s_out,
                    scales=dict(p=s_p, u=s_u, u2=s_u2, c=s_c, s=s_s, d=s_d, out=s_out))


def row_mask(slots: int, g: int) -> np.ndarray:
    m = np.zeros(slots)
    m[::g] = 1.0
    return m


# ---------------------------------------------------------------- trainer
class FusedTrainer:
    """Encrypted enhanced-NAG logistic regression on one GPU.

    Packing: each block is m x g (m rows, g = S/m columns); a batch is
    ``blocks_per_batch`` consecutive row blocks (the BASELINE paper shape
    packs a 1,024-row batch as 8 blocks of 128 x 256); ``cols`` column
    blocks cover the f+1 coefficients.  Mini-batch mode visits one batch
    per iteration in order; full-batch mode sums every batch's gradient
    before one B̄ product and update (enctrain.py:356-359, 374-381).

    Every iteration reads its batch in place from the HBM-resident
    encrypted dataset (one captured CUDA graph per phase, re-pointed at the
    next batch with ``helr_nag_graph_update``), or, when ``host_stream`` is
    set, from two staging buffers filled by host-to-device copies.
    """

    def __init__(self, ctx: GpuContext, ds, rows_per_block: int, blocks_per_batch: int = 1,
                 mode: str = "mini_batch", poly: PolyApprox = BASELINE_CUBIC, schedule=None,
                 epsilon: float = 1e-8, enhanced: bool = True, use_graph: bool = False, bsgs: bool = True,
                 refresh_bits: int = 47, bsgs_bits: Optional[int] = None, rows_bits: Optional[int] = None,
                 shard: tuple = (0, 1), reducer=None, device_encode: bool = True):
        if mode not in ("mini_batch", "full_batch"):
            raise ValueError(f"mode must be mini_batch or full_batch, got {mode!r}")
        from .optimizer import ExpDecay
        self.ctx = ctx
        self.ck = ctx.ckks
        self.ds = ds
        self.mode = mode
        self.poly = poly
        self.schedule = schedule if schedule is not None else ExpDecay()
        self.epsilon = epsilon
        self.enhanced = enhanced
        self.use_graph = use_graph
        # full-batch sharding (shard.py): this rank's batches, and the in-place
        # SUM of the raw gradient residues across ranks (None: single rank)
        self.shard_rank, self.shard_world = int(shard[0]), int(shard[1])
        if self.shard_world > 1 and mode != "full_batch":
            raise ValueError("only the full-batch gradient shards; mini-batch runs replicas")
        if self.shard_world > 1 and reducer is None:
            raise ValueError("a sharded trainer needs a reducer (shard.ResidueAllReduce)")
        self.reducer = reducer
        # client-side encoding on the device (helr_encode; encoder.py is the
        # host twin, kept for comparisons)
        self.device_encode = device_encode
        # W, V re-enter each iteration at scale 2^refresh_bits: above Delta = 2^40
        # so the refresh's fresh encryption noise is negligible, below 2^50 so
        # the row-start mask still encodes at >= 2^35
        self.refresh_bits = refresh_bits
        # bootstrap='ckks' contexts (real bootstrapping, bootstrap.py): the sine
        # of EvalMod is linear only for |message| << q_0, so W', V' reach the
        # bottom level two bits lower (q_0 / scale = 2^12), and the refreshed
        # W, V come back at the working top's canonical scale
        self.real_bootstrap = getattr(ctx, "bootstrap_mode", "refresh") == "ckks"
        self.out_bits = OUT_SCALE_BITS - 2 if self.real_bootstrap else OUT_SCALE_BITS
        if self.real_bootstrap:
            self.refresh_bits = ctx.ckks.scale_bits
        self.layout: BlockLayout = plan_layout(ds.n_samples, ds.n_features, ctx.params, rows_per_block)
        lay = self.layout
        self.rows = blocks_per_batch
        self.cols = lay.col_blocks
        self.n_batches = -(-lay.row_blocks // blocks_per_batch)
        self.log_g = int(math.log2(lay.g))
        self.log_m = int(math.log2(lay.m))
        self.batch_rows = lay.m * blocks_per_batch
        # sum_col_vec halves and sum_rows as grouped hoisted rotate-and-sums
        # (groups of at most log_baby / log_baby_rows bits; 0 = one key switch
        # per power-of-two rotation)
        if not bsgs:
            self.log_baby = self.log_baby_rows = 0
        else:
            self.log_baby = (self.log_g + 1) // 2 if bsgs_bits is None else bsgs_bits
            self.log_baby_rows = (self.log_m + 1) // 2 if rows_bits is None else rows_bits
            if not (0 <= self.log_baby <= 5 and 0 <= self.log_baby_rows <= 5):
                raise ValueError("hoisted groups hold at most 31 rotations: group bits must be in [0, 5]")
            if self.log_g == 0:
                self.log_baby = 0
            if self.log_m == 0:
                self.log_baby_rows = 0
        self.qpoly = poly.complement().padded(3)
        self.lib = _lib.load()
        _bind(self.lib)
        self._graphs: dict = {}
        self._warm = False
        # graph capture is not allowed on the legacy default stream
        self.stream = torch.cuda.Stream(device=ctx.device)
        self.timings: dict = {}
        self.host_stream = False
        self.z_host = None
        self.b_host = None
        self.copy_stream = None
        self._d2h_ev = None
        self._prepare()

    # ------------------------------------------------------------ client side
    def _prepare(self):
        ctx, ck, lay, ds = self.ctx, self.ck, self.layout, self.ds
        t0 = time.perf_counter()
        Z = ds.X * ds.y[:, None]
        blocks = pack_matrix_array(Z, lay)                       # (row_blocks, cols, S)
        nb, R, C = self.n_batches, self.rows, self.cols
        top = ck.top_level
        s_top = ck.level_scales[top]
        L, N = ck.L, ck.n
        self.z = torch.empty((nb, R, C, 2, L, N), dtype=torch.int64, device=ctx.device)
        zflat = self.z.view(nb * R * C, 2, L, N)
        nblk = lay.row_blocks * C
        flat = blocks.reshape(nblk, ck.slots)
        chunk = 64
        encode = ctx.encode_slots if self.device_encode else ctx.encoder.encode
        for s in range(0, nblk, chunk):
            coef = encode(flat[s:s + chunk], s_top)
            ctx.encrypt_to(coef, zflat[s:s + coef.shape[0]], top)
        if nb * R * C > nblk:  # zero blocks padding the last batch (encryptions of 0)
            pad = nb * R * C - nblk
            ctx.encrypt_to(np.zeros((pad, N), dtype=np.int64), zflat[nblk:], top)
        self.s_z = s_top
        # B̄ per batch (mini) or merged over batches (full), from the real rows
        # of each batch (enctrain.py:132-142; BASELINE: "computed per batch")
        self.scalers = []
        for b in range(nb):
            lo = b * self.batch_rows
            hi = min(lo + self.batch_rows, ds.n_samples)
            self.scalers.append(scaler_for(ds.X[lo:hi], self.epsilon))
        vecs = [merge_bbar(self.scalers).b] if self.mode == "full_batch" else [s.b for s in self.scalers]
        bb = np.stack([np.stack(replicate_rows(v, lay)) for v in vecs])   # (nbb, C, S)
        self.bbar = torch.empty((bb.shape[0], C, 2, L, N), dtype=torch.int64, device=ctx.device)
        bflat = bb.reshape(-1, ck.slots)
        bout = self.bbar.view(-1, 2, L, N)
        # B̄ entries are small (1e-3 per 1,024-row batch, ~1e-5 merged over the
        # whole dataset); encode them at s_top / max|B̄| so the encryption noise
        # stays ~2^-30 relative to B̄ (the planner tracks the exact scale)
        # B̄'s fixed encryption noise is a per-batch relative error of the
        # preconditioner that the NAG dynamics amplify over the whole run
        # (tools/precision_probe.py: 7.5e-10 relative -> 7e-7 of weight error
        # after 1,239 Paper-mini iterations), so B̄ is encrypted up to 2^6 above
        # s_top / max|B̄| — as far as the NAG constants that multiply the
        # product G * B̄ stay >= 2^33 (relative rounding <= 2^-34)
        s_b0 = s_top / float(np.max(np.abs(bb)))
        trial = plan_iteration(ck, top, 2.0 ** self.refresh_bits, 2.0 ** self.refresh_bits, s_top, s_b0, self.qpoly,
                               1.0, 0.37, self.out_bits)
        ca_bits = math.log2(min(abs(trial.ints[5]), abs(trial.ints[8])))
        self.bbar_extra_bits = int(max(0, min(BBAR_EXTRA_BITS, math.floor(ca_bits - 33))))
        self.s_b = s_b0 * 2.0 ** self.bbar_extra_bits
        for s in range(0, bflat.shape[0], chunk):
            coef = encode(bflat[s:s + chunk], self.s_b)
            ctx.encrypt_to(coef, bout[s:s + coef.shape[0]], top)
        # W0 = V0 = enc(0) at the top level (enctrain.py:145-151)
        self.wv = torch.empty((2 * C, 2, L, N), dtype=torch.int64, device=ctx.device)
        ctx.encrypt_to(np.zeros((2 * C, N), dtype=np.int64), self.wv, top)
        self.wv_tmp = torch.empty_like(self.wv)
        self.level = top
        self.s_w = self.s_v = s_top
        self.alpha0 = ALPHA0_INIT
        self.alpha1 = next_alpha(ALPHA0_INIT)
        self.t = 0
        # keys: left/right 2^i (sum_col_vec), g*2^i (sum_rows)
        S = ck.slots
        if self.log_baby > 0:
            steps = [k for grp in grouped_steps(self.log_g, self.log_baby) for k in grp]
        else:
            steps = [1 << i for i in range(self.log_g)]
        if self.log_baby_rows > 0:
            rsteps = [k for grp in grouped_steps(self.log_m, self.log_baby_rows, lay.g) for k in grp]
        else:
            rsteps = [lay.g << i for i in range(self.log_m)]
        self.gal_left = [pow(5, k, 2 * N) for k in steps]
        self.gal_right = [pow(5, S - k, 2 * N) for k in steps]
        self.gal_rows = [pow(5, k % S, 2 * N) for k in rsteps]
        keys = lambda gs: (ctypes.c_void_p * max(1, len(gs)))(*[ctx.galois_key(g).data_ptr() for g in gs])
        self._k_left, self._k_right, self._k_rows = keys(self.gal_left), keys(self.gal_right), keys(self.gal_rows)
        self._masks: dict = {}
        self.consts_dev = torch.zeros((NCONST, L), dtype=torch.int64, device=ctx.device)
        # ring of pinned host buffers: an async H2D copy must never read a host
        # buffer that a later iteration has already overwritten
        self._cring = [torch.zeros((NCONST, L), dtype=torch.int64).pin_memory() for _ in range(4)]
        self._cev = [None] * len(self._cring)
        self._ci = 0
        self.grad = torch.empty((C, 2, L, N), dtype=torch.int64, device=ctx.device)
        self.w_host = torch.empty((2 * C, 2, L, N), dtype=torch.int64).pin_memory()
        torch.cuda.synchronize()
        self.timings["prepare_s"] = time.perf_counter() - t0

    def enable_host_stream(self):
        """Keep the encrypted dataset in pinned host memory and stream each
        batch to the device inside the iteration (the e2e path).

        Copies are double-buffered on a separate copy stream: while iteration
        t runs on staging buffer t % 2, the host-to-device copy of the next
        batch fills the other buffer (event-ordered both ways), so the PCIe
        transfer overlaps the encrypted arithmetic."""
        if self.z_host is None:
            self.z_host = torch.empty(self.z.shape, dtype=torch.int64, pin_memory=True)
            self.z_host.copy_(self.z)
            self.b_host = torch.empty(self.bbar.shape, dtype=torch.int64, pin_memory=True)
            self.b_host.copy_(self.bbar)
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(device=self.ctx.device)
            self._zst = [torch.empty_like(self.z[0]) for _ in range(2)]
            self._bst = [torch.empty_like(self.bbar[0]) for _ in range(2)]
            self.w_snap = torch.empty_like(self.wv)
        self._d2h_ev = None
        self._buf = 0
        self._loaded = [None, None]   # (batch, bbar index) each buffer holds / is receiving
        self._ready = [None, None]    # copy finished (copy stream)
        self._free = [None, None]     # last reader finished (compute stream)
        self.host_stream = True

    def disable_host_stream(self):
        self.host_stream = False

    def bytes_per_step(self) -> tuple:
        """(H2D, D2H) bytes a host-streamed mini-batch step moves."""
        cs = self.wv[0].numel() * 8
        h2d = (self.rows * self.cols + self.cols) * cs + NCONST * self.ck.L * 8
        active = (self.level_after_next() + 1) * self.ck.n * 8 * 2
        d2h = 2 * self.cols * active
        return h2d, d2h

    def level_after_next(self) -> int:
        lvl = self.level if self.level >= ITER_DEPTH else self.ck.top_level
        return lvl - ITER_DEPTH

    def _mask(self, lw: int, scale: float) -> torch.Tensor:
        key = (lw, round(scale))
        if key not in self._masks:
            ck = self.ck
            coef = self.ctx.encoder.encode(row_mask(ck.slots, self.layout.g), scale)
            self._masks[key] = self.ctx._plain(coef, lw - 1)
        return self._masks[key]

    # ------------------------------------------------------------ iteration
    def step_scalars(self, t: int, gamma_rows: int):
        lr = lr_at(self.schedule, t)
        eta = (1.0 - self.alpha0) / self.alpha1
        gamma = lr / gamma_rows if self.enhanced else lr / self.ds.n_samples
        mult = (1.0 + gamma) if self.enhanced else gamma
        return lr, eta, gamma, mult

    def _refresh_if_needed(self) -> bool:
        # bootstrap_policy (enctrain.py:242-255): refresh when the next
        # iteration cannot fit; one iteration consumes ITER_DEPTH limbs.
        if self.level >= ITER_DEPTH:
            return False
        self.refresh()
        return True

    def refresh(self):
        """Bring W and V back to the working top: real CKKS bootstrapping of
        the 2C ciphertexts in one batched circuit when the context was made
        with bootstrap='ckks' (bootstrap.Bootstrapper, evaluation keys only),
        else the refresh stand-in (NOT bootstrapping; see helr_refresh)."""
        ck = self.ck
        if self.real_bootstrap:
            if abs(self.s_w / self.s_v - 1.0) > 1e-12:
                raise ValueError("W and V must share a scale to bootstrap as one batch")
            out, lvl, scale = self.ctx.bootstrap_batch(self.wv, self.level, self.s_w)
            self.ctx.counters["bootstrap"] += self.wv.shape[0]
            self.wv.copy_(out)
            self.level = lvl
            self.s_w = self.s_v = scale
            return
        top = ck.top_level
        target = float(2 ** self.refresh_bits)
        ratio = target / self.s_w
        first = self.ctx._take_ct_ids(self.wv.shape[0])
        stream = torch.cuda.current_stream().cuda_stream
        self.ctx._call("helr_refresh", self.ctx.sk.data_ptr(), self.wv.data_ptr(), self.level, float(ratio),
                       self.wv_tmp.data_ptr(), top, self.wv.shape[0], self.ctx.enc_seed, first, stream)
        self.wv.copy_(self.wv_tmp)
        self.level = top
        self.s_w = self.s_v = target

    def _args(self, plan: IterPlan, phase: int, zb) -> NagArgs:
        C = self.cols
        cs = self.wv[0].numel() * 8
        z_ptr, b_ptr = zb
        return NagArgs(z=z_ptr, rows=self.rows, cols=C, log_g=self.log_g, log_m=self.log_m,
                       w=self.wv.data_ptr(), v=self.wv.data_ptr() + C * cs, bbar=b_ptr,
                       lw=plan.lw, rlk=self.ctx.rlk.data_ptr(), rot_left=self._k_left, rot_right=self._k_right,
                       rot_rows=self._k_rows, mask_pt=self._mask(plan.lw, plan.mask_scale).data_ptr(),
                       consts=self.consts_dev.data_ptr(), grad=self.grad.data_ptr(), phase=phase,
                       log_baby=self.log_baby, log_baby_rows=self.log_baby_rows)

    def _upload_consts(self, plan: IterPlan):
        i = self._ci
        self._ci = (i + 1) % len(self._cring)
        if self._cev[i] is not None:
            self._cev[i].synchronize()
        buf = self._cring[i]
        buf.copy_(torch.from_numpy(plan.consts.view(np.int64)))
        self.consts_dev.copy_(buf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._cev[i] = ev

    def _stage(self, batch: int, bbar_index: int, with_bbar: bool = True):
        """Make (batch, bbar_index) resident in a staging buffer; returns the
        (z, bbar) device pointers the iteration reads."""
        if not self.host_stream:
            # resident dataset: the iteration reads the batch in place (a
            # captured graph is re-pointed with helr_nag_graph_update)
            return self.z[batch].data_ptr(), self.bbar[bbar_index].data_ptr()
        buf = self._buf
        if self._loaded[buf] is None or self._loaded[buf][0] != batch or self._loaded[buf][1] != bbar_index:
            self._prefetch(buf, batch, bbar_index)
        self.stream.wait_event(self._ready[buf])
        return self._zst[buf].data_ptr(), self._bst[buf].data_ptr()

    def _prefetch(self, buf: int, batch: int, bbar_index: int):
        cs = self.copy_stream
        if self._free[buf] is not None:
            cs.wait_event(self._free[buf])
        prev = self._loaded[buf]
        with torch.cuda.stream(cs):
            self._zst[buf].copy_(self.z_host[batch], non_blocking=True)
            if prev is None or prev[1] != bbar_index:
                self._bst[buf].copy_(self.b_host[bbar_index], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._ready[buf] = ev
        self._loaded[buf] = (batch, bbar_index)

    def _release(self, next_batch: int, next_bbar: int):
        """The current buffer's reader is enqueued: mark it, flip buffers and
        start copying the next batch into the other one."""
        buf = self._buf
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self._free[buf] = ev
        self._buf = 1 - buf
        self._prefetch(self._buf, next_batch, next_bbar)

    def _run(self, args: NagArgs):
        stream = torch.cuda.current_stream().cuda_stream
        if not self.use_graph or not self._warm:
            # eager; the first eager run also allocates the driver workspace
            _lib.check(self.lib.helr_nag_iteration(self.ctx.handle, ctypes.byref(args), stream), "helr_nag_iteration")
            self._warm = True
            return
        # host-streamed batches alternate between two staging buffers: one
        # graph each; resident batches share one graph re-pointed per step
        ptrs = (args.z, args.bbar)
        key = (args.lw, args.phase, args.mask_pt) + (ptrs if self.host_stream else ())
        ent = self._graphs.get(key)
        if ent is None:
            g = ctypes.c_void_p()
            _lib.check(self.lib.helr_nag_graph_capture(self.ctx.handle, ctypes.byref(args), stream, ctypes.byref(g)),
                       "helr_nag_graph_capture")
            ent = self._graphs[key] = [g, ptrs]
        elif ent[1] != ptrs:
            _lib.check(self.lib.helr_nag_graph_update(self.ctx.handle, ctypes.byref(args), stream, ent[0]),
                       "helr_nag_graph_update")
            ent[1] = ptrs
        _lib.check(self.lib.helr_nag_graph_launch(ent[0], stream), "helr_nag_graph_launch")

    def profile_iteration(self, batch: Optional[int] = None) -> dict:
        """One iteration replayed from a freshly captured graph whose kernels are
        bracketed by the library's category events (helr_prof_*), so the
        per-category device times carry no host launch gaps."""
        lib = self.lib
        lib.helr_prof_enable.argtypes = [ctypes.c_int]
        saved, self._graphs = self._graphs, {}
        use, self.use_graph = self.use_graph, True
        warm, self._warm = self._warm, True
        lib.helr_prof_enable(1)
        try:
            info = self.iterate(batch)
        finally:
            lib.helr_prof_enable(0)
            for g, _ in self._graphs.values():
                torch.cuda.synchronize()
                lib.helr_nag_graph_destroy(g)
            self._graphs, self.use_graph, self._warm = saved, use, warm
        return info

    def iterate(self, batch: Optional[int] = None) -> dict:
        """One NAG iteration (mini-batch: batch ``t mod n_batches``; full: all),
        issued on the trainer's stream."""
        with torch.cuda.stream(self.stream):
            return self._iterate(batch)

    def _iterate(self, batch: Optional[int]) -> dict:
        refreshed = self._refresh_if_needed()
        if self.mode == "mini_batch":
            b = (self.t % self.n_batches) if batch is None else batch
            gamma_rows = min(self.batch_rows, self.ds.n_samples - b * self.batch_rows)
        else:
            b = 0
            gamma_rows = self.ds.n_samples
        lr, eta, gamma, mult = self.step_scalars(self.t, gamma_rows)
        plan = plan_iteration(self.ck, self.level, self.s_w, self.s_v, self.s_z, self.s_b, self.qpoly, mult, eta,
                              self.out_bits)
        self._upload_consts(plan)
        nbt = self.n_batches
        if self.mode == "mini_batch":
            zb = self._stage(b, b)
            self._run(self._args(plan, 0, zb))
            if self.host_stream:
                self._release((b + 1) % nbt, (b + 1) % nbt)
        else:
            mine = partition(nbt, self.shard_rank, self.shard_world)
            zb = None
            for i, bb in enumerate(mine):
                zb = self._stage(bb, 0, with_bbar=(i == 0))
                self._run(self._args(plan, 1 if i == 0 else 2, zb))
                if self.host_stream:
                    self._release(mine[(i + 1) % len(mine)], 0)
            if zb is None:  # more ranks than batches: this rank contributes zero
                self.grad.zero_()
                zb = self._stage(0, 0)
            if self.shard_world > 1:
                self.combine_gradient()
            self._run(self._args(plan, 3, zb))
            if self.host_stream:  # the finish phase reads the last buffer's B̄ too
                ev = torch.cuda.Event()
                ev.record(self.stream)
                self._free[1 - self._buf] = ev
        level_start = self.level
        self.level -= ITER_DEPTH
        self.s_w = self.s_v = plan.s_out
        self.alpha0, self.alpha1 = self.alpha1, next_alpha(self.alpha1)
        self.t += 1
        if self.host_stream:
            # the step's result leaves the device: the updated weight ciphertexts
            lv = self.level + 1
            self._read_back(lv)
        return dict(iteration=self.t, lr=lr, eta=eta, gamma=gamma, level_start=level_start,
                    level_after=self.level, refreshed=refreshed)

    def _read_back(self, lv: int):
        """The step's result leaves the device off the critical path: a
        device-side snapshot of the active W, V limbs (one contiguous copy per
        polynomial, on the compute stream), then its device-to-host copy on
        the copy stream, overlapping the next iteration.  The snapshot is
        rewritten only after the previous read-back has finished."""
        if self._d2h_ev is not None:
            self.stream.wait_event(self._d2h_ev)
        for ci in range(self.wv.shape[0]):
            for pi in range(2):
                self.w_snap[ci, pi, :lv].copy_(self.wv[ci, pi, :lv], non_blocking=True)
        ready = torch.cuda.Event()
        ready.record(self.stream)
        cs = self.copy_stream
        cs.wait_event(ready)
        with torch.cuda.stream(cs):
            for ci in range(self.wv.shape[0]):
                for pi in range(2):
                    self.w_host[ci, pi, :lv].copy_(self.w_snap[ci, pi, :lv], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._d2h_ev = ev

    def finish_host_stream(self):
        """Order the compute stream after the last weight read-back (call
        before recording the end of a timed e2e region)."""
        if self._d2h_ev is not None:
            self.stream.wait_event(self._d2h_ev)

    def combine_gradient(self):
        """Sum the ranks' partial gradients (raw residue words, exact in 63
        bits) and fold them back to canonical residues on the device."""
        self.reducer(self.grad)
        lv = self.level - 5  # the gradient's level (helr_nag_args.grad)
        self.ctx._call("helr_reduce", self.grad.data_ptr(), self.grad.data_ptr(), self.cols, lv,
                       torch.cuda.current_stream().cuda_stream)

    # ------------------------------------------------------------ readout
    def weights(self) -> np.ndarray:
        """Decrypt W and read row 0 of each column block (decode_weights,
        enctrain.py:266-289, without the exact replication check)."""
        ctx, lay = self.ctx, self.layout
        C = self.cols
        with torch.cuda.stream(self.stream):
            out = torch.empty((C, self.ck.n), dtype=torch.int64, device=ctx.device)
            ctx._call("helr_decrypt", ctx.sk.data_ptr(), self.wv.data_ptr(), C, self.level, out.data_ptr(),
                      self.stream.cuda_stream)
            if self.device_encode:
                slots = ctx.decode_coefficients(out, self.s_w)
            else:
                slots = ctx.encoder.decode(out.cpu().numpy(), self.s_w)
        segs = []
        for j in range(C):
            grid = slots[j].reshape(lay.m, lay.g)
            segs.append(np.real(grid[0]))
        return np.concatenate(segs)[: lay.cols]

    def close(self):
        torch.cuda.synchronize(self.ctx.device)
        for g, _ in self._graphs.values():
            self.lib.helr_nag_graph_destroy(g)
        self._graphs.clear()
