// ctx.cu — context creation: ring tables, basis-conversion constants,
// workspace; thread-local error reporting for the C ABI.
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/helr_ckks.h"
#include "ctx.cuh"

typedef unsigned __int128 h128;

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
// Clear an error left by an earlier, unrelated runtime call on this thread so
// it is not blamed on the next launch; report it once on stderr.
void clear_stale_error(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[helr] stale CUDA error before %s: %s\n", where, cudaGetErrorString(e));
}

bool cuda_ok(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return false;
}

extern "C" int helr_last_error(char* buf, size_t len) {
    if (!buf || !len) return (int)g_err.size();
    size_t m = g_err.size() < len - 1 ? g_err.size() : len - 1;
    memcpy(buf, g_err.data(), m);
    buf[m] = 0;
    return (int)g_err.size();
}

extern "C" int helr_version(void) { return 100; }

// ---- host modular helpers -------------------------------------------------
static u64 hmul(u64 a, u64 b, u64 q) { return (u64)(((h128)a * b) % q); }
static u64 hpow(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = hmul(r, b, q);
        b = hmul(b, b, q);
        e >>= 1;
    }
    return r;
}
static u64 hinv(u64 a, u64 q) { return hpow(a % q, q - 2, q); }
static u64 hshoup(u64 w, u64 q) { return (u64)(((h128)w << 64) / q); }
static unsigned hbrv(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

// ModUp table layout for (level l, digit j) at modup_off[l*beta + j]:
//   [ns] hinv, [ns] hinv_sh, [ns][nt] hmod, [ns][nt] hmod_sh
// with ns = source limbs of the digit, nt = targets (l+1-ns) + K, targets in
// extended order e = 0..l+K excluding the digit's own limbs.
static void modup_entry(helr_ctx* c, int l, int j, std::vector<u64>& out) {
    const int nl = l + 1, al = c->alpha;
    const int lo = j * al, hi = (lo + al < nl) ? lo + al : nl;
    const int ns = hi - lo;
    std::vector<int> tgt;
    for (int e = 0; e < nl + c->K; e++) {
        if (e >= lo && e < hi) continue;
        tgt.push_back(e < nl ? e : c->L + (e - nl));
    }
    const int nt = (int)tgt.size();
    std::vector<u64> hv(ns), hvs(ns), hm((size_t)ns * nt), hms((size_t)ns * nt);
    for (int k = 0; k < ns; k++) {
        u64 sk = c->primes[lo + k], prod = 1;
        for (int k2 = 0; k2 < ns; k2++)
            if (k2 != k) prod = hmul(prod, c->primes[lo + k2] % sk, sk);
        hv[k] = hinv(prod, sk);
        hvs[k] = hshoup(hv[k], sk);
        for (int t = 0; t < nt; t++) {
            u64 qt = c->primes[tgt[t]], p2 = 1;
            for (int k2 = 0; k2 < ns; k2++)
                if (k2 != k) p2 = hmul(p2, c->primes[lo + k2] % qt, qt);
            hm[(size_t)k * nt + t] = p2;
            hms[(size_t)k * nt + t] = hshoup(p2, qt);
        }
    }
    out.insert(out.end(), hv.begin(), hv.end());
    out.insert(out.end(), hvs.begin(), hvs.end());
    out.insert(out.end(), hm.begin(), hm.end());
    out.insert(out.end(), hms.begin(), hms.end());
}

size_t ks_workspace_words(const helr_ctx* c, int batch) {
    // per item at the top level: INTT copy (L) + modup (beta*(L+K)) +
    // accumulators (2*(L+K)) + ModDown conversions (2*L) + tensor (3*L)
    const size_t per = (size_t)c->L + (size_t)c->beta * c->LK + 2 * (size_t)c->LK + 2 * (size_t)c->L + 3 * (size_t)c->L;
    return per * c->n * (size_t)batch;
}

extern "C" int helr_ctx_create(helr_ctx** out, int log_n, int L, int K, int dnum, const uint64_t* primes,
                               const uint64_t* psi, int cbd_eta, int max_batch) {
    if (!out || !primes || !psi) { set_error("null argument"); return HELR_EINVAL; }
    if (log_n < 2 || log_n > 17) { set_error("log_n must be in [2, 17]"); return HELR_EINVAL; }
    if (L < 2 || K < 1 || L + K > HELR_MAXP) { set_error("bad prime counts"); return HELR_EINVAL; }
    if (dnum < 1 || dnum > L) { set_error("bad dnum"); return HELR_EINVAL; }
    const int alpha = (L + dnum - 1) / dnum;
    if (max_batch < 1) max_batch = 1;
    const int n = 1 << log_n;
    for (int i = 0; i < L + K; i++) {
        // < 2^61: lazy NTT values in [0, 8q) and 128-bit key-product sums of
        // up to 63 terms must fit their words
        if (primes[i] >= (1ull << 61) || (primes[i] - 1) % (2ull * n) != 0) {
            set_error("primes must be < 2^61 and = 1 mod 2N");
            return HELR_EINVAL;
        }
        if (hpow(psi[i], (u64)n, primes[i]) != primes[i] - 1) {
            set_error("psi is not a primitive 2N-th root");
            return HELR_EINVAL;
        }
    }
    helr_ctx* c = new helr_ctx();
    c->log_n = log_n; c->n = n; c->L = L; c->K = K; c->LK = L + K; c->dnum = dnum; c->alpha = alpha;
    c->beta = (L + alpha - 1) / alpha; c->eta = cbd_eta; c->max_batch = max_batch;
    c->primes.assign(primes, primes + L + K);
    c->psi.assign(psi, psi + L + K);
    const int LK = L + K;

    // ---- build every table on the host, one contiguous upload -----------
    std::vector<u64> h;
    auto put = [&](size_t words) { size_t o = (h.size() + 1) & ~(size_t)1; h.resize(o + words); return o; };  // 16-byte aligned
    size_t o_q = put(LK), o_b1 = put(LK), o_b0 = put(LK);
    // twiddles as interleaved (w, floor(w 2^64 / q)) pairs: one 16-byte load per butterfly group
    size_t o_tw = put(2 * (size_t)LK * n);
    size_t o_itw = put(2 * (size_t)LK * n);
    size_t o_ni = put(LK), o_nis = put(LK), o_i1 = put(LK), o_i1s = put(LK);
    size_t o_one = put(LK), o_t128 = put(LK), o_t128s = put(LK);  // floor(2^64/q); 2^128 mod q (+ Shoup)
    // fp64 twiddles / constants (bit patterns of doubles) for the fp64 NTT path
    size_t o_twd = put((size_t)LK * n), o_itwd = put((size_t)LK * n);
    size_t o_qd = put(LK), o_qinvd = put(LK), o_nid = put(LK), o_i1d = put(LK);
    auto dbits = [](double v) { u64 b; memcpy(&b, &v, 8); return b; };
    for (int p = 0; p < LK; p++) {
        u64 q = primes[p];
        h[o_q + p] = q;
        h[o_one + p] = hshoup(1, q);
        {
            u64 t64 = (u64)(((h128)1 << 64) % q);
            u64 t = hmul(t64, t64, q);
            h[o_t128 + p] = t;
            h[o_t128s + p] = hshoup(t, q);
        }
        h128 ratio = (~(h128)0) / q;  // floor((2^128 - 1)/q) == floor(2^128/q) for odd q
        h[o_b1 + p] = (u64)(ratio >> 64);
        h[o_b0 + p] = (u64)ratio;
        u64 ip = hinv(psi[p], q);
        std::vector<u64> pw(n), ipw(n);
        pw[0] = 1; ipw[0] = 1;
        for (int k = 1; k < n; k++) { pw[k] = hmul(pw[k - 1], psi[p], q); ipw[k] = hmul(ipw[k - 1], ip, q); }
        for (int k = 0; k < n; k++) {
            unsigned e = hbrv((unsigned)k, log_n);
            u64 w = pw[e], iw = ipw[e];
            h[o_tw + 2 * ((size_t)p * n + k)] = w;
            h[o_tw + 2 * ((size_t)p * n + k) + 1] = hshoup(w, q);
            h[o_itw + 2 * ((size_t)p * n + k)] = iw;
            h[o_itw + 2 * ((size_t)p * n + k) + 1] = hshoup(iw, q);
            h[o_twd + (size_t)p * n + k] = dbits((double)w);
            h[o_itwd + (size_t)p * n + k] = dbits((double)iw);
        }
        u64 ni = hinv((u64)n, q);
        h[o_ni + p] = ni;
        h[o_nis + p] = hshoup(ni, q);
        u64 i1 = hmul(h[o_itw + 2 * ((size_t)p * n + 1)], ni, q);
        h[o_i1 + p] = i1;
        h[o_i1s + p] = hshoup(i1, q);
        h[o_qd + p] = dbits((double)q);
        h[o_qinvd + p] = dbits(1.0 / (double)q);
        h[o_nid + p] = dbits((double)ni);
        h[o_i1d + p] = dbits((double)i1);
    }
    // rescale constants
    size_t o_ql = put((size_t)L * L), o_qls = put((size_t)L * L);
    for (int l = 1; l < L; l++)
        for (int i = 0; i < l; i++) {
            u64 v = hinv(primes[l] % primes[i], primes[i]);
            h[o_ql + (size_t)l * L + i] = v;
            h[o_qls + (size_t)l * L + i] = hshoup(v, primes[i]);
        }
    // ModDown constants
    size_t o_phi = put(K), o_phis = put(K), o_phm = put((size_t)K * L), o_phms = put((size_t)K * L);
    size_t o_pi = put(L), o_pis = put(L), o_pm = put(L), o_pms = put(L), o_pid = put(K);
    for (int k = 0; k < K; k++) {
        u64 pk = primes[L + k], prod = 1;
        for (int k2 = 0; k2 < K; k2++)
            if (k2 != k) prod = hmul(prod, primes[L + k2] % pk, pk);
        h[o_phi + k] = hinv(prod, pk);
        h[o_phis + k] = hshoup(h[o_phi + k], pk);
        for (int i = 0; i < L; i++) {
            u64 qi = primes[i], p2 = 1;
            for (int k2 = 0; k2 < K; k2++)
                if (k2 != k) p2 = hmul(p2, primes[L + k2] % qi, qi);
            h[o_phm + (size_t)k * L + i] = p2;
            h[o_phms + (size_t)k * L + i] = hshoup(p2, qi);
        }
    }
    for (int i = 0; i < L; i++) {
        u64 qi = primes[i], pm = 1;
        for (int k = 0; k < K; k++) pm = hmul(pm, primes[L + k] % qi, qi);
        h[o_pm + i] = pm;
        h[o_pms + i] = hshoup(pm, qi);
        h[o_pi + i] = hinv(pm, qi);
        h[o_pis + i] = hshoup(h[o_pi + i], qi);
    }
    for (int k = 0; k < K; k++) {  // 1/p_k as IEEE double bits (centred ModDown)
        double inv = 1.0 / (double)primes[L + k];
        memcpy(&h[o_pid + k], &inv, sizeof(double));
    }
    // Merged ModDown + rescale by M_l = P * q_l (level l >= 1), source basis
    // {p_0..p_{K-1}, q_l} -> Q_{l-1}.  Per level, at mr_off[l]:
    //   [K+1] hinv, [K+1] hinv_sh, [K+1][L] hmod, [K+1][L] hmod_sh,
    //   [L] M mod q_i, [L] M mod q_i shoup, [L] M^-1 mod q_i, [L] M^-1 shoup, [K+1] 1/m_k (double bits)
    c->mr_off.assign((size_t)L, 0);
    for (int l = 1; l < L; l++) {
        const int ns = K + 1;
        std::vector<u64> src(ns);
        for (int k = 0; k < K; k++) src[k] = primes[L + k];
        src[K] = primes[l];
        std::vector<u64> e(2 * ns + 2 * (size_t)ns * L + 4 * (size_t)L + ns, 0);
        u64* hv = e.data();
        u64* hvs = hv + ns;
        u64* hm = hvs + ns;
        u64* hms = hm + (size_t)ns * L;
        u64* mm = hms + (size_t)ns * L;
        u64* mms = mm + L;
        u64* mi = mms + L;
        u64* mis = mi + L;
        u64* dinv = mis + L;
        for (int k = 0; k < ns; k++) {
            u64 sk = src[k], prod = 1;
            for (int k2 = 0; k2 < ns; k2++)
                if (k2 != k) prod = hmul(prod, src[k2] % sk, sk);
            hv[k] = hinv(prod, sk);
            hvs[k] = hshoup(hv[k], sk);
            double inv = 1.0 / (double)sk;
            memcpy(&dinv[k], &inv, sizeof(double));
            for (int i = 0; i < l; i++) {
                u64 qi = primes[i], p2 = 1;
                for (int k2 = 0; k2 < ns; k2++)
                    if (k2 != k) p2 = hmul(p2, src[k2] % qi, qi);
                hm[(size_t)k * L + i] = p2;
                hms[(size_t)k * L + i] = hshoup(p2, qi);
            }
        }
        for (int i = 0; i < l; i++) {
            u64 qi = primes[i], m = 1;
            for (int k = 0; k < ns; k++) m = hmul(m, src[k] % qi, qi);
            mm[i] = m;
            mms[i] = hshoup(m, qi);
            mi[i] = hinv(m, qi);
            mis[i] = hshoup(mi[i], qi);
        }
        size_t o = put(e.size());
        memcpy(&h[o], e.data(), e.size() * sizeof(u64));
        c->mr_off[l] = o;
    }
    // X^(N/2) in NTT form per ciphertext prime (imul)
    size_t o_im = put((size_t)L * n);
    for (int p = 0; p < L; p++)
        for (int k = 0; k < n; k++) {
            u64 e = ((2ull * hbrv((unsigned)k, log_n) + 1) * (u64)(n / 2)) % (2ull * n);
            h[o_im + (size_t)p * n + k] = hpow(psi[p], e, primes[p]);
        }
    // ModUp constants per (level, digit)
    c->modup_off.assign((size_t)L * c->beta, 0);
    for (int l = 0; l < L; l++) {
        const int nd = (l + 1 + alpha - 1) / alpha;
        for (int j = 0; j < nd; j++) {
            std::vector<u64> e;
            modup_entry(c, l, j, e);
            size_t o = put(e.size());
            memcpy(&h[o], e.data(), e.size() * sizeof(u64));
            c->modup_off[(size_t)l * c->beta + j] = o;
        }
    }

    c->tab_words = h.size();
    if (!cuda_ok(cudaMalloc(&c->d_tab, h.size() * sizeof(u64)), "cudaMalloc(tables)")) { delete c; return HELR_ECUDA; }
    if (!cuda_ok(cudaMemcpy(c->d_tab, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice), "upload tables")) {
        cudaFree(c->d_tab); delete c; return HELR_ECUDA;
    }
    const u64* d = c->d_tab;
    auto dp = [&](size_t o) { return reinterpret_cast<const double*>(d + o); };
    c->t = Tables{d + o_q, d + o_b1, d + o_b0, d + o_tw, d + o_itw,
                  d + o_ni, d + o_nis, d + o_i1, d + o_i1s, log_n, n, L, K, alpha, c->beta,
                  dp(o_twd), dp(o_itwd), dp(o_qd), dp(o_qinvd), dp(o_nid), dp(o_i1d)};
    c->qlinv = d + o_ql; c->qlinv_sh = d + o_qls;
    c->md_phinv = d + o_phi; c->md_phinv_sh = d + o_phis;
    c->md_phmod = d + o_phm; c->md_phmod_sh = d + o_phms;
    c->md_pinv = d + o_pi; c->md_pinv_sh = d + o_pis; c->pmod = d + o_pm; c->pmod_sh = d + o_pms; c->md_pinv_dbl = d + o_pid;
    c->imul_f = d + o_im;
    c->one_sh = d + o_one; c->t128 = d + o_t128; c->t128_sh = d + o_t128s;
    c->modup = d;  // offsets in modup_off are absolute word offsets into d_tab

    if (!cuda_ok(cudaMalloc(&c->d_modup_offs, c->modup_off.size() * sizeof(size_t)), "cudaMalloc(offsets)") ||
        !cuda_ok(cudaMemcpy(c->d_modup_offs, c->modup_off.data(), c->modup_off.size() * sizeof(size_t),
                            cudaMemcpyHostToDevice), "upload offsets")) {
        cudaFree(c->d_tab); delete c; return HELR_ECUDA;
    }
    c->ws_words = ks_workspace_words(c, max_batch);
    if (!cuda_ok(cudaMalloc(&c->ws, c->ws_words * sizeof(u64)), "cudaMalloc(workspace)")) {
        cudaFree(c->d_tab); delete c; return HELR_ENOMEM;
    }
    *out = c;
    return HELR_OK;
}

extern "C" int helr_ctx_destroy(helr_ctx* c) {
    if (!c) return HELR_OK;
    cudaFree(c->d_tab);
    cudaFree(c->d_modup_offs);
    cudaFree(c->ws);
    cudaFree(c->nag_ws);
    cudaFree(c->enc_tw);
    cudaFree(c->enc_tpos);
    cudaFree(c->enc_tneg);
    delete c;
    return HELR_OK;
}
