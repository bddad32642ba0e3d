// nag.cu — fused enhanced-NAG iteration: the reference's loop body
// (enctrain.py:344-398: enc_gradient 162-197, enc_quad_gradient 200-208,
// enc_nag_update 211-239) as one native call over a whole batch.
//
// Differences from the literal reference circuit (same values in exact
// arithmetic):
//  - depth 7 instead of 9: q1 u and q0 land directly on the level of
//    u^2 * (q3 u); the three NAG constant products fold into two linear
//    combinations followed by one rescale;
//  - sum_rows runs once on the batch total instead of once per row block
//    (rotations are linear), and the batch total itself is one tensor sum
//    followed by one relinearisation;
//  - the row blocks of a batch move through every rotation stage together,
//    so each Galois key is streamed once per stage for the whole batch.
#include <cuda_runtime.h>

#include <vector>

#include "../../include/helr_ckks.h"
#include "ops_internal.cuh"

#define TRY(x)                 \
    do {                       \
        int _r = (x);          \
        if (_r) return _r;     \
    } while (0)

// The driver workspace belongs to the context (like the key-switching
// workspace).  It only grows, and never while a captured graph that points
// into it is alive (helr_nag_graph_capture / _destroy keep the count): a
// reallocation would leave those graphs writing freed memory.  One fused
// trainer per context at a time: trainers on different streams would race
// on this scratch.
static int nag_buffers(helr_ctx* c, int rows, int cols, cudaStream_t s, u64** out) {
    const size_t cs = 2ull * c->L * c->n;
    const size_t need = cs * (7ull * rows + 5ull * cols);
    if (c->nag_ws && c->nag_words >= need) { *out = c->nag_ws; return HELR_OK; }
    cudaStreamCaptureStatus st;
    if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
        set_error("nag workspace must be allocated before graph capture (run one iteration first)");
        return HELR_EINVAL;
    }
    if (c->nag_graphs > 0) {
        set_error("nag workspace would grow while captured graphs still use it (destroy them first)");
        return HELR_EINVAL;
    }
    if (c->nag_ws) {
        cudaStreamSynchronize(s);
        cudaFree(c->nag_ws);
        c->nag_ws = nullptr;
        c->nag_words = 0;
    }
    if (!cuda_ok(cudaMalloc(&c->nag_ws, need * sizeof(u64)), "cudaMalloc(nag workspace)")) return HELR_ENOMEM;
    c->nag_words = need;
    *out = c->nag_ws;
    return HELR_OK;
}

// opaque graph handle returned to the host: the exec plus its context
struct nag_graph {
    cudaGraphExec_t exec;
    helr_ctx* ctx;
};

static long long pow_mod_ll(long long b, long long e, long long m) {
    long long r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = (long long)((__int128)r * b % m);
        b = (long long)((__int128)b * b % m);
        e >>= 1;
    }
    return r;
}

extern "C" int helr_rotsum_groups(int log_total, int max_bits, int* bits) {
    if (log_total <= 0 || max_bits <= 0) return 0;
    const int ng = (log_total + max_bits - 1) / max_bits;
    const int base = log_total / ng, rem = log_total % ng;
    for (int j = 0; j < ng && j < 64; j++) bits[j] = base + (j < rem ? 1 : 0);
    return ng;
}

// out = sum_{k < 2^log_total} rot(in, sign * stride * k) as grouped hoisted
// rotate-and-sums (helr_rotsum_groups): group j sums rotations
// stride * k * 2^off_j, k = 1..2^bits_j - 1, plus the identity, with one ModUp
// and one ModDown per group.  keys: group 0's keys, then group 1's, ...
// `tmp` is scratch; `out` may alias `in`, neither may alias `tmp`.
static int grouped_rotsum(helr_ctx* c, const uint64_t* const* keys, int log_total, int max_bits, int sign,
                          long long stride, const u64* in, u64* out, u64* tmp, int R, int level, cudaStream_t s) {
    const long long CS = 2ll * c->L * c->n, two_n = 2ll * c->n, slots = c->n / 2;
    int bits[64];
    const int ng = helr_rotsum_groups(log_total, max_bits, bits);
    if (ng == 0) {
        if (out != in) cudaMemcpyAsync(out, in, (size_t)R * CS * sizeof(u64), cudaMemcpyDeviceToDevice, s);
        return HELR_OK;
    }
    // ping-pong so that the last group writes `out`
    const u64* src = in;
    int off = 0, kbase = 0;
    for (int j = 0; j < ng; j++) {
        u64* dst = ((ng - 1 - j) % 2 == 0) ? out : tmp;
        if (dst == src) dst = (dst == out) ? tmp : out;  // never alias a group's input
        const int nk = (1 << bits[j]) - 1;
        if (nk > HELR_MAX_HOIST) {
            set_error("grouped rotsum: at most 5 bits (31 rotations) per hoisted group");
            return HELR_EINVAL;
        }
        long long gal[HELR_MAX_HOIST];
        for (int k = 1; k <= nk; k++) {
            const long long step = ((stride * (long long)k) << off) % slots;
            gal[k - 1] = pow_mod_ll(5, sign > 0 ? step : (slots - step) % slots, two_n);
        }
        TRY(op_rotsum_hoisted(c, src, CS, nk, gal, (const u64* const*)(keys + kbase), dst, CS, R, level, 1, s));
        src = dst;
        off += bits[j];
        kbase += nk;
    }
    if (src != out) cudaMemcpyAsync(out, src, (size_t)R * CS * sizeof(u64), cudaMemcpyDeviceToDevice, s);
    return HELR_OK;
}

static int nag_run(helr_ctx* c, const helr_nag_args* a, cudaStream_t s) {
    const int L = c->L, n = c->n;
    const long long CS = 2ll * L * n;
    const int R = a->rows, C = a->cols, lw = a->lw;
    const long long two_n = 2ll * n, slots = n / 2;
    if (a->log_g + a->log_m != c->log_n - 1) { set_error("nag: m*g must equal N/2"); return HELR_EINVAL; }
    if (R < 1 || C < 1) { set_error("nag: rows and cols must be >= 1"); return HELR_EINVAL; }
    if (a->phase < 0 || a->phase > 3) { set_error("nag: bad phase"); return HELR_EINVAL; }
    if (lw < 7 || lw >= L) { set_error("nag: lw must be in [7, L)"); return HELR_EINVAL; }

    u64* ws = nullptr;
    TRY(nag_buffers(c, R, C, s, &ws));
    u64* T1 = ws;                        // [R] products before rescale
    u64* X0 = T1 + (size_t)R * CS;       // [R] ping
    u64* X1 = X0 + (size_t)R * CS;       // [R] pong
    u64* U = X1 + (size_t)R * CS;        // [R] u            (lw-2)
    u64* U2 = U + (size_t)R * CS;        // [R] u^2          (lw-3)
    u64* TQ = U2 + (size_t)R * CS;       // [R] q3 u         (lw-3)
    u64* QU = TQ + (size_t)R * CS;       // [R] poly(u)      (lw-4)
    u64* G = QU + (size_t)R * CS;        // [C] gradient     (lw-5)
    u64* GT = G + (size_t)C * CS;        // [C] temp
    u64* D = GT + (size_t)C * CS;        // [C] G*Bbar       (lw-6)
    u64* NW = D + (size_t)C * CS;        // [C] W' before rescale
    u64* NV = NW + (size_t)C * CS;       // [C] V' before rescale
    const u64* K = a->consts;
    auto kc = [&](int idx) { return K + (size_t)idx * L; };

    if (a->phase != 3) {
        // 1) P_r = relin(sum_j Z_rj (x) W_j), rescale -> lw-1
        TRY(op_mul_relin_rescale_sum(c, a->z, (long long)C * CS, CS, a->w, 0, CS, C, a->rlk, X0, CS, R, lw, s));
        // 2) sum_{k<g} rot(P, k): the left half of sum_col_vec (hesim.py:255-257)
        u64* cur = X0;
        u64* nxt = X1;
        if (a->log_baby > 0) {
            TRY(grouped_rotsum(c, a->rot_left, a->log_g, a->log_baby, +1, 1, cur, nxt, T1, R, lw - 1, s));
            u64* t = cur; cur = nxt; nxt = t;
        } else {
            for (int i = 0; i < a->log_g; i++) {
                const long long g = pow_mod_ll(5, 1ll << i, two_n);
                TRY(op_rotate(c, cur, CS, g, a->rot_left[i], nxt, CS, R, lw - 1, 1, s));
                u64* t = cur; cur = nxt; nxt = t;
            }
        }
        // 3) row-start mask (hesim.py:258-260), rescale -> lw-2
        TRY(op_ew(c, EW_MULPT, cur, CS, a->mask_pt, 0, T1, CS, R, lw - 1, s));
        TRY(op_rescale(c, T1, CS, cur, CS, R, lw - 1, s));
        // 4) sum_{k<g} rot(M, -k): the right half (hesim.py:262-264)
        if (a->log_baby > 0) {
            TRY(grouped_rotsum(c, a->rot_right, a->log_g, a->log_baby, -1, 1, cur, U, T1, R, lw - 2, s));
        } else {
            for (int i = 0; i < a->log_g; i++) {
                const long long g = pow_mod_ll(5, slots - (1ll << i), two_n);
                u64* dst = (i == a->log_g - 1) ? U : nxt;
                TRY(op_rotate(c, cur, CS, g, a->rot_right[i], dst, CS, R, lw - 2, 1, s));
                u64* t = cur; cur = dst; nxt = t;
            }
            if (a->log_g == 0) {
                cudaMemcpyAsync(U, cur, (size_t)R * CS * sizeof(u64), cudaMemcpyDeviceToDevice, s);
            }
        }
        // 5) u^2 (lw-3)
        TRY(op_mul_relin_rescale_sum(c, U, CS, 0, U, CS, 0, 1, a->rlk, U2, CS, R, lw - 2, s));
        // 6) q3 u (lw-3)
        TRY(op_ew(c, EW_MULC, U, CS, kc(0), 0, T1, CS, R, lw - 2, s));
        TRY(op_rescale(c, T1, CS, TQ, CS, R, lw - 2, s));
        // 7) u^2 * (q3 u) (lw-4)
        TRY(op_mul_relin_rescale_sum(c, U2, CS, 0, TQ, CS, 0, 1, a->rlk, QU, CS, R, lw - 3, s));
        // 8) + q1 u + q2 u^2 landing on lw-4, + q0
        {
            const u64* xs[2] = {U, U2};
            const long long ss[2] = {CS, CS};
            const u64* ks[2] = {kc(1), kc(2)};
            TRY(op_lincomb(c, 2, xs, ss, ks, T1, CS, R, lw - 3, s));  // U read at its lower limbs
            TRY(op_rescale(c, T1, CS, X0, CS, R, lw - 3, s));
            TRY(op_ew(c, EW_ADD, QU, CS, X0, CS, QU, CS, R, lw - 4, s));
            TRY(op_ew(c, EW_ADDC, QU, CS, kc(3), 0, QU, CS, R, lw - 4, s));
        }
        // 9) G_j = rescale(relin(sum_r QU_r (x) Z_rj))  (lw-5)
        u64* Gdst = (a->phase == 2) ? GT : (a->phase == 1 ? a->grad : G);
        TRY(op_mul_relin_rescale_sum(c, QU, 0, CS, a->z, CS, (long long)C * CS, R, a->rlk, Gdst, CS, C, lw - 4, s));
        if (a->phase == 2) TRY(op_ew(c, EW_ADD, a->grad, CS, GT, CS, a->grad, CS, C, lw - 5, s));
        if (a->phase != 0) return HELR_OK;
    }
    const u64* Gsrc = (a->phase == 3) ? a->grad : G;
    // 10) sum_rows: rotate-and-add by g, 2g, ..., (m/2) g (hesim.py:278-280)
    if (a->log_baby_rows > 0) {
        TRY(grouped_rotsum(c, a->rot_rows, a->log_m, a->log_baby_rows, +1, 1ll << a->log_g, Gsrc, G, GT, C, lw - 5,
                           s));
    } else {
        const u64* cur = Gsrc;
        u64* bufs[2] = {GT, D};
        for (int i = 0; i < a->log_m; i++) {
            const long long g = pow_mod_ll(5, (1ll << a->log_g) << i, two_n);
            u64* dst = bufs[i & 1];
            TRY(op_rotate(c, cur, CS, g, a->rot_rows[i], dst, CS, C, lw - 5, 1, s));
            cur = dst;
        }
        if (cur != G) cudaMemcpyAsync(G, cur, (size_t)C * CS * sizeof(u64), cudaMemcpyDeviceToDevice, s);
    }
    // 11) D_j = G_j * Bbar_j (enc_quad_gradient, enctrain.py:200-208), lw-6
    TRY(op_mul_relin_rescale_sum(c, G, CS, 0, a->bbar, CS, 0, 1, a->rlk, D, CS, C, lw - 5, s));
    // 12) NAG (enctrain.py:211-239):  V' = W + (1+g) D,  W' = (1-e) V' + e V
    {
        const u64* xv[2] = {a->w, D};
        const long long sv[2] = {CS, CS};
        const u64* kv[2] = {kc(4), kc(5)};
        TRY(op_lincomb(c, 2, xv, sv, kv, NV, CS, C, lw - 6, s));
        const u64* xw[3] = {a->w, a->v, D};
        const long long sw[3] = {CS, CS, CS};
        const u64* kw[3] = {kc(6), kc(7), kc(8)};
        TRY(op_lincomb(c, 3, xw, sw, kw, NW, CS, C, lw - 6, s));
        TRY(op_rescale(c, NV, CS, a->v, CS, C, lw - 6, s));
        TRY(op_rescale(c, NW, CS, a->w, CS, C, lw - 6, s));
    }
    return HELR_OK;
}

extern "C" int helr_nag_iteration(helr_ctx* c, const helr_nag_args* a, void* stream) {
    clear_stale_error("helr_nag_iteration");
    if (!c || !a) { set_error("null argument"); return HELR_EINVAL; }
    return nag_run(c, a, (cudaStream_t)stream);
}

extern "C" int helr_nag_graph_capture(helr_ctx* c, const helr_nag_args* a, void* stream, void** graph_exec) {
    clear_stale_error("helr_nag_graph_capture");
    if (!c || !a || !graph_exec) { set_error("null argument"); return HELR_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    u64* ws = nullptr;
    TRY(nag_buffers(c, a->rows, a->cols, s, &ws));
    if (!cuda_ok(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture")) return HELR_ECUDA;
    int r = nag_run(c, a, s);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (r) { if (graph) cudaGraphDestroy(graph); return r; }
    if (!cuda_ok(e, "end capture")) return HELR_ECUDA;
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (!cuda_ok(e, "graph instantiate")) return HELR_ECUDA;
    nag_graph* h = new nag_graph{exec, c};
    c->nag_graphs++;
    *graph_exec = (void*)h;
    return HELR_OK;
}

// Re-point a captured iteration at new arguments (a different batch of the
// resident dataset, other constants) without a new instantiation: capture
// the iteration again and update the executable graph in place (the
// topology is identical for equal (rows, cols, lw, phase, group bits), so
// cudaGraphExecUpdate only rewrites kernel parameters).  This replaces a
// per-step device-to-device copy of the batch into fixed staging buffers.
extern "C" int helr_nag_graph_update(helr_ctx* c, const helr_nag_args* a, void* stream, void* graph_exec) {
    clear_stale_error("helr_nag_graph_update");
    if (!c || !a || !graph_exec) { set_error("null argument"); return HELR_EINVAL; }
    nag_graph* h = (nag_graph*)graph_exec;
    if (h->ctx != c) { set_error("graph belongs to another context"); return HELR_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    if (!cuda_ok(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture")) return HELR_ECUDA;
    int r = nag_run(c, a, s);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (r) { if (graph) cudaGraphDestroy(graph); return r; }
    if (!cuda_ok(e, "end capture")) return HELR_ECUDA;
    cudaGraphExecUpdateResultInfo info;
    e = cudaGraphExecUpdate(h->exec, graph, &info);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("graph update failed: topology changed");
        return HELR_EINVAL;
    }
    return HELR_OK;
}

extern "C" int helr_nag_graph_launch(void* graph_exec, void* stream) {
    clear_stale_error("helr_nag_graph_launch");
    if (!graph_exec) { set_error("null graph"); return HELR_EINVAL; }
    nag_graph* h = (nag_graph*)graph_exec;
    if (!cuda_ok(cudaGraphLaunch(h->exec, (cudaStream_t)stream), "graph launch")) return HELR_ECUDA;
    return HELR_OK;
}

extern "C" int helr_nag_graph_destroy(void* graph_exec) {
    clear_stale_error("helr_nag_graph_destroy");
    if (graph_exec) {
        nag_graph* h = (nag_graph*)graph_exec;
        cudaGraphExecDestroy(h->exec);
        if (h->ctx && h->ctx->nag_graphs > 0) h->ctx->nag_graphs--;
        delete h;
    }
    return HELR_OK;
}
