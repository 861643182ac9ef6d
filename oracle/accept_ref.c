/* Oracle: tree acceptance (greedy and rejection sampling) — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, sequential C written from the paper and the readings in DESIGN.md. It is built
 * by oracle/accept.py (gcc -O2 -ffp-contract=off, no fast-math) and called through ctypes
 * by tests/ and bench.py's cpu_baseline leg only. It shares no code with the CUDA path.
 *
 * Paper: "speculative tokens are fed into the LLM to be verified in a single decoding step
 * ... If the speculative tokens from the SSM are consistent with LLM, the LLM accepts these
 * tokens" and speculative decoding "is consistent with the distribution of autoregressive
 * decoding"; tree-based verification. The paper gives no acceptance rule;
 * DESIGN.md readings Z5-Z8, Z15 fix it:
 *   GREEDY        walk from the root; accept the child whose token equals argmax of the
 *                 target row (ties -> lowest vocab id; duplicate sibling tokens -> lowest
 *                 node index); bonus = argmax at the last accepted node.
 *   SAMPLE_DELTA  children visited in ascending node index; child x accepted w.p.
 *                 min(1, p(x)/1) (draft q = one-hot); on rejection p <- norm(p with p(x)=0);
 *                 bonus ~ residual p.
 *   SAMPLE_MSS    children drawn i.i.d. from q_c (draft_probs row c): accept w.p.
 *                 min(1, p(x)/q(x)); on rejection p <- norm(max(p - q, 0)). q_c is read only
 *                 for a node that HAS children (reading Z29: a node without children has no
 *                 distribution its children were drawn from; its draft row is never used).
 * Arithmetic: distributions are unsigned integer weights
 *   w_v = trunc(exp_spec((l_v - max l) * inv_tau) * 2^32), all sums/compares in integers,
 *   uniforms are word 0 of Philox4x32-10(counter=(trial, node, lo32(step), lo32(gid)),
 *   key=(lo32(seed), hi32(seed))), trial = child rank for child tests, 0xFFFFFFFF for the bonus.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <math.h>

typedef unsigned __int128 u128;

enum { MODE_GREEDY = 0, MODE_DELTA = 1, MODE_MSS = 2 };
enum { FLAG_MALFORMED = 1, FLAG_NONFINITE = 2 };
#define MAX_TREE 64

/* ---- Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) ---- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint32_t uniform_word(uint64_t seed, uint64_t step, int64_t gid, uint32_t trial, uint32_t node) {
    uint32_t ctr[4] = {trial, node, (uint32_t)step, (uint32_t)(uint64_t)gid};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[0];
}

/* ---- exp_spec: fixed-sequence fp32 exp for x <= 0 ----
 * Every operation is a single IEEE-754 binary32 round-to-nearest-even operation, in this
 * order, with no fused multiply-add (built with -ffp-contract=off). */
float oracle_exp_spec(float x) {
    if (!(x >= -32.0f)) return 0.0f;   /* also NaN; exp(-32) * 2^32 < 1 -> weight 0 */
    const float LOG2E = 1.44269502735137939453125f;  /* 0x3FB8AA3B */
    const float C1 = 0.693359375f;                    /* 0x3F318000 */
    const float C2 = -2.12194440e-4f;                 /* 0xB95E8083 */
    float t = x * LOG2E;
    float n = rintf(t);                /* round half to even (default rounding mode) */
    float a = n * C1;                  /* exact: C1 has 9 significant bits, |n| <= 47 */
    float r = x - a;
    float b = n * C2;
    r = r - b;
    float p = 1.9875691500e-4f;
    p = p * r; p = p + 1.3981999507e-3f;
    p = p * r; p = p + 8.3334519073e-3f;
    p = p * r; p = p + 4.1665795894e-2f;
    p = p * r; p = p + 1.6666665459e-1f;
    p = p * r; p = p + 5.0000001201e-1f;
    float z = r * r;
    float y = p * z;
    y = y + r;
    y = y + 1.0f;
    return ldexpf(y, (int)n);
}

static float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static float logit_at(const void* logits, int is_bf16, int64_t row, int V, int v) {
    if (is_bf16) return bf16_to_f32(((const uint16_t*)logits)[row * (int64_t)V + v]);
    return ((const float*)logits)[row * (int64_t)V + v];
}

/* Target weights of one row: w_v = trunc(ldexp(exp_spec((l_v - m) * inv_tau), 32)). Returns
 * -1 if the row has a non-finite logit, else 0; *Z = sum of weights. */
int oracle_row_weights(const void* logits, int is_bf16, int64_t row, int V, float inv_tau,
                       uint64_t* w, uint64_t* Z) {
    float m = -INFINITY;
    for (int v = 0; v < V; ++v) {
        float l = logit_at(logits, is_bf16, row, V, v);
        if (!isfinite(l)) return -1;
        if (l > m) m = l;
    }
    uint64_t z = 0;
    for (int v = 0; v < V; ++v) {
        float l = logit_at(logits, is_bf16, row, V, v);
        float x = l - m;
        x = x * inv_tau;
        float e = oracle_exp_spec(x);
        w[v] = (uint64_t)ldexpf(e, 32);      /* exact scaling; conversion truncates */
        z += w[v];
    }
    *Z = z;
    return 0;
}

/* Draft weights qw_v = trunc(ldexp(q_v, 32)). */
static uint64_t draft_weights(const float* q, int64_t row, int V, uint64_t* qw) {
    uint64_t z = 0;
    for (int v = 0; v < V; ++v) {
        float qv = q[row * (int64_t)V + v];
        qw[v] = (qv > 0.0f) ? (uint64_t)ldexpf(qv, 32) : 0;
        z += qw[v];
    }
    return z;
}

static int bitlen128(u128 x) {
    int n = 0;
    while (x) { ++n; x >>= 1; }
    return n;
}

/* Smallest v with sum_{j<=v} w_j > t. */
static int inverse_cdf(const uint64_t* w, int V, uint64_t t) {
    uint64_t acc = 0;
    for (int v = 0; v < V; ++v) {
        acc += w[v];
        if (acc > t) return v;
    }
    return V - 1;
}

static int greedy_argmax(const void* logits, int is_bf16, int64_t row, int V, int* nonfinite) {
    int best = 0;
    float bv = -INFINITY;
    *nonfinite = 0;
    for (int v = 0; v < V; ++v) {
        float l = logit_at(logits, is_bf16, row, V, v);
        if (!isfinite(l)) { *nonfinite = 1; return -1; }
        if (l > bv) { bv = l; best = v; }   /* strict: ties keep the lowest id */
    }
    return best;
}

/* draft_row (MSS, may be NULL = identity): row of draft_probs holding node i's q (global node
 * index i); a node with children whose draft_row is negative makes the tree malformed. */
int oracle_tree_accept_rows(int mode, const void* logits, int logits_is_bf16, const float* draft_probs,
                            const int32_t* draft_row, const int32_t* parent, const int32_t* token,
                            const int32_t* tree_off, const int64_t* gid, int B, int V, float temperature,
                            uint64_t seed, uint64_t step, int32_t* accepted_len, int32_t* path, int32_t* bonus,
                            int32_t* flags) {
    float inv_tau = 1.0f / temperature;
    uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * V);
    uint64_t* w_saved = (uint64_t*)malloc(sizeof(uint64_t) * V);
    uint64_t* qw = (uint64_t*)malloc(sizeof(uint64_t) * V);
    u128* r = (u128*)malloc(sizeof(u128) * V);
    for (int b = 0; b < B; ++b) {
        int off = tree_off[b], T = tree_off[b + 1] - tree_off[b];
        int32_t* pth = path + (int64_t)b * MAX_TREE;
        for (int k = 0; k < MAX_TREE; ++k) pth[k] = -1;
        accepted_len[b] = 0;
        bonus[b] = -1;
        flags[b] = 0;
        /* tree validation (reading Z1): 1 <= T <= 64, parent[0] = -1, 0 <= parent[i] < i, and
         * every draft node's token is a vocabulary id, 0 <= token[i] < V for i >= 1 (the root's
         * token is the last committed one and is never tested) */
        int ok = (T >= 1 && T <= MAX_TREE && parent[off] == -1);
        for (int i = 1; ok && i < T; ++i)
            ok = (parent[off + i] >= 0 && parent[off + i] < i && token[off + i] >= 0 && token[off + i] < V);
        /* MSS with a row map: every node with children needs a draft row */
        for (int i = 1; ok && mode == MODE_MSS && draft_row && i < T; ++i)
            ok = draft_row[off + parent[off + i]] >= 0;
        if (!ok) { flags[b] = FLAG_MALFORMED; continue; }

        int c = 0, a = 0;
        pth[0] = 0;
        for (;;) {
            int64_t row = off + c;
            int nch = 0, ch[MAX_TREE];
            for (int x = c + 1; x < T; ++x)
                if (parent[off + x] == c) ch[nch++] = x;   /* ascending node index */
            int next = -1;
            if (mode == MODE_GREEDY) {
                int nf;
                int t = greedy_argmax(logits, logits_is_bf16, row, V, &nf);
                if (nf) { flags[b] |= FLAG_NONFINITE; break; }
                for (int k = 0; k < nch; ++k)
                    if (token[off + ch[k]] == t) { next = ch[k]; break; }
                if (next < 0) { bonus[b] = t; break; }
            } else {
                uint64_t Z;
                if (oracle_row_weights(logits, logits_is_bf16, row, V, inv_tau, w, &Z) != 0) {
                    flags[b] |= FLAG_NONFINITE;
                    break;
                }
                uint64_t Zq = 0;
                if (mode == MODE_MSS && nch > 0) {   /* reading Z29: leaves' rows are not read */
                    const int64_t qrow = draft_row ? draft_row[off + c] : row;
                    /* the draft row must be a probability vector: every q_v in [0, 1] (reading
                     * Z15 extended: otherwise the sample is flagged like a non-finite row) */
                    int okq = 1;
                    for (int v = 0; v < V && okq; ++v) {
                        float qv = draft_probs[qrow * (int64_t)V + v];
                        okq = (qv >= 0.0f && qv <= 1.0f);
                    }
                    if (!okq) { flags[b] |= FLAG_NONFINITE; break; }
                    Zq = draft_weights(draft_probs, qrow, V, qw);
                }
                for (int k = 0; k < nch; ++k) {
                    int x = ch[k];
                    int tk = token[off + x];
                    uint32_t U = uniform_word(seed, step, gid[b], (uint32_t)k, (uint32_t)c);
                    int acc;
                    if (mode == MODE_DELTA) {
                        acc = ((u128)U * Z) < ((u128)w[tk] << 32);
                    } else if (qw[tk] == 0) {
                        acc = w[tk] > 0;
                    } else {
                        acc = ((u128)U * ((u128)qw[tk] * Z)) < (((u128)w[tk] * Zq) << 32);
                    }
                    if (acc) { next = x; break; }
                    /* rejection: residual distribution */
                    if (mode == MODE_DELTA) {
                        Z -= w[tk];
                        w[tk] = 0;
                    } else {
                        memcpy(w_saved, w, sizeof(uint64_t) * V);
                        uint64_t Z_saved = Z;
                        u128 mx = 0;
                        for (int v = 0; v < V; ++v) {
                            u128 lhs = (u128)w[v] * Zq, rhs = (u128)qw[v] * Z;
                            r[v] = lhs > rhs ? lhs - rhs : 0;
                            if (r[v] > mx) mx = r[v];
                        }
                        int s = bitlen128(mx) - 32;
                        if (s < 0) s = 0;
                        Z = 0;
                        for (int v = 0; v < V; ++v) { w[v] = (uint64_t)(r[v] >> s); Z += w[v]; }
                        if (Z == 0) {   /* degenerate residual (quantisation only): keep prior */
                            memcpy(w, w_saved, sizeof(uint64_t) * V);
                            Z = Z_saved;
                        }
                    }
                }
                if (next < 0) {
                    uint32_t U2 = uniform_word(seed, step, gid[b], 0xFFFFFFFFu, (uint32_t)c);
                    uint64_t t = (uint64_t)(((u128)U2 * Z) >> 32);
                    bonus[b] = inverse_cdf(w, V, t);
                    break;
                }
            }
            c = next;
            ++a;
            pth[a] = c;
        }
        accepted_len[b] = a;
    }
    free(w); free(w_saved); free(qw); free(r);
    return 0;
}

int oracle_tree_accept(int mode, const void* logits, int logits_is_bf16, const float* draft_probs,
                       const int32_t* parent, const int32_t* token, const int32_t* tree_off,
                       const int64_t* gid, int B, int V, float temperature, uint64_t seed,
                       uint64_t step, int32_t* accepted_len, int32_t* path, int32_t* bonus,
                       int32_t* flags) {
    return oracle_tree_accept_rows(mode, logits, logits_is_bf16, draft_probs, NULL, parent, token, tree_off, gid,
                                   B, V, temperature, seed, step, accepted_len, path, bonus, flags);
}

/* Elementwise exp_spec over an array (for pin tests that sweep many inputs). */
void oracle_exp_spec_array(const float* x, float* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = oracle_exp_spec(x[i]);
}
