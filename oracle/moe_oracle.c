/*
 * moe_oracle.c — CPU oracle for the MoE-layer hot path (see moe_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for tests/, smoke() and bench.py's
 * CPU-baseline leg. Never linked into or called by the product library.
 *
 * Every function cites the reference lines it restates. The routing maps
 * are restated with a different algorithm (stable counting sort instead of
 * std::stable_sort) so that agreement with oracle/_ref (the reference's own
 * code) is evidence, not tautology.
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* routing                                                              */
/* ------------------------------------------------------------------ */

/* routing.cpp:113-131: capacity = ceil(cf*T*k/n) in double; loads start as
 * the full per-group slot counts; scan t = T-1..0; a token whose groups
 * include ANY group with load > capacity is dropped whole and decrements
 * all of its groups. Group of expert e = e / (E/n) (routing.cpp:44-47). */
/* Thread count of the dense fp32 parts (the host process may inherit
 * OMP_NUM_THREADS=1 from a launcher; the CPU baseline sets it explicitly). */
void orc_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
int orc_get_threads(void) { return omp_get_max_threads(); }

int orc_capacity_drop(int64_t T, int64_t E, int64_t k, int64_t n_groups, double cf,
                      const int32_t* experts, uint8_t* dropped) {
    if (T < 0 || E < 1 || k < 1 || n_groups < 1 || E % n_groups != 0 || !(cf > 0.0)) return -2;
    const int64_t per = E / n_groups;
    const int64_t capacity =
        (int64_t)ceil(cf * (double)T * (double)k / (double)n_groups);
    int64_t* load = (int64_t*)calloc((size_t)n_groups, sizeof(int64_t));
    for (int64_t i = 0; i < T * k; ++i) load[experts[i] / per]++;
    for (int64_t t = T - 1; t >= 0; --t) {
        int over = 0;
        for (int64_t j = 0; j < k; ++j)
            if (load[experts[t * k + j] / per] > capacity) over = 1;
        dropped[t] = (uint8_t)over;
        if (over)
            for (int64_t j = 0; j < k; ++j) load[experts[t * k + j] / per]--;
    }
    free(load);
    return 0;
}

/* routing.cpp:135-187. Entries (t, slot) of non-dropped tokens whose expert
 * is in [my_rank*E/n, (my_rank+1)*E/n) are ordered by (expert, source_rank,
 * token) stably; row_map_in = t*k + slot. per_expert_counts counts every
 * retained (t, slot) over ALL experts (routing.cpp:158). Restated as a
 * counting sort over bins (expert_local * n + source_rank): a pass in
 * (t, slot) order is stable, and within one token the k experts are
 * distinct so the order is total. */
int64_t orc_build_scatter_map(int64_t T, int64_t E, int64_t k, const int32_t* experts,
                              const int32_t* source_rank, const uint8_t* dropped,
                              int64_t n, int64_t my_rank, int64_t* row_map_in,
                              int64_t* per_expert_counts, int32_t* out_expert,
                              int32_t* out_source_rank) {
    if (n < 1 || my_rank < 0 || my_rank >= n || E % n != 0) return -2;
    const int64_t el = E / n;
    const int64_t first = my_rank * el;
    /* source ranks in the reference tests are arbitrary ints; bin them by
     * their rank order. Determine the distinct range. */
    int32_t smin = 0, smax = 0;
    for (int64_t t = 0; t < T; ++t) {
        if (t == 0 || source_rank[t] < smin) smin = source_rank[t];
        if (t == 0 || source_rank[t] > smax) smax = source_rank[t];
    }
    const int64_t ns = (int64_t)smax - smin + 1;
    const int64_t nbins = el * ns;
    int64_t* cnt = (int64_t*)calloc((size_t)nbins + 1, sizeof(int64_t));
    for (int64_t e = 0; e < E; ++e) per_expert_counts[e] = 0;
    for (int64_t t = 0; t < T; ++t) {
        if (dropped[t]) continue;
        for (int64_t j = 0; j < k; ++j) {
            const int32_t e = experts[t * k + j];
            per_expert_counts[e]++;
            if (e >= first && e < first + el) cnt[(e - first) * ns + (source_rank[t] - smin) + 1]++;
        }
    }
    for (int64_t b = 0; b < nbins; ++b) cnt[b + 1] += cnt[b];
    const int64_t rows = cnt[nbins];
    for (int64_t t = 0; t < T; ++t) {
        if (dropped[t]) continue;
        for (int64_t j = 0; j < k; ++j) {
            const int32_t e = experts[t * k + j];
            if (e < first || e >= first + el) continue;
            const int64_t pos = cnt[(e - first) * ns + (source_rank[t] - smin)]++;
            row_map_in[pos] = t * k + j;
            out_expert[pos] = e;
            out_source_rank[pos] = source_rank[t];
        }
    }
    free(cnt);
    return rows;
}

/* routing.cpp:189-217: per expert run, tiles of tile_rows rows; dependent
 * ranks = distinct source ranks of the tile's rows (ascending, since rows are
 * sorted by source rank within an expert). */
int64_t orc_sort_tokens_for_tiles(int64_t rows, const int32_t* out_expert,
                                  const int32_t* out_source_rank, int64_t tile_rows,
                                  int32_t* tile_expert, int64_t* tile_begin,
                                  int64_t* tile_end, uint64_t* tile_rank_mask) {
    if (tile_rows < 1) return -2;
    int64_t nt = 0, row = 0;
    while (row < rows) {
        const int32_t e = out_expert[row];
        int64_t end = row;
        while (end < rows && out_expert[end] == e) end++;
        for (int64_t b = row; b < end; b += tile_rows) {
            const int64_t te = (b + tile_rows < end) ? b + tile_rows : end;
            uint64_t mask = 0;
            for (int64_t r = b; r < te; ++r) mask |= 1ull << out_source_rank[r];
            tile_expert[nt] = e;
            tile_begin[nt] = b;
            tile_end[nt] = te;
            tile_rank_mask[nt] = mask;
            nt++;
        }
        row = end;
    }
    return nt;
}

/* routing.cpp:219-262. */
int orc_balance_metrics(int64_t T, int64_t E, int64_t k, const int32_t* experts,
                        const uint8_t* dropped, int64_t n, int64_t* per_group_load,
                        double* loss, int64_t* capacity, double* drop_rate) {
    if (n < 1 || E % n != 0) return -2;
    const int64_t per = E / n;
    int64_t* assigned = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    int64_t ndrop = 0;
    for (int64_t g = 0; g < n; ++g) per_group_load[g] = 0;
    for (int64_t t = 0; t < T; ++t) {
        if (dropped[t]) ndrop++;
        for (int64_t j = 0; j < k; ++j) {
            const int64_t g = experts[t * k + j] / per;
            assigned[g]++;
            if (!dropped[t]) per_group_load[g]++;
        }
    }
    int64_t tl = 0, ta = 0;
    for (int64_t g = 0; g < n; ++g) { tl += per_group_load[g]; ta += assigned[g]; }
    double l = 0.0;
    if (tl > 0 && ta > 0) {
        for (int64_t g = 0; g < n; ++g)
            l += ((double)per_group_load[g] / (double)tl) * ((double)assigned[g] / (double)ta);
        l *= (double)n;
    }
    *loss = l;
    *capacity = T > 0 ? (int64_t)ceil((double)T * (double)k / (double)n) : 0;
    *drop_rate = T > 0 ? (double)ndrop / (double)T : 0.0;
    free(assigned);
    return 0;
}

/* ------------------------------------------------------------------ */
/* numerics                                                             */
/* ------------------------------------------------------------------ */

/* numerics.cpp:29-68. Restated with ilogb/ldexp/rint (RNE) rather than the
 * reference's frexp/nearbyint. */
double orc_round_to(int fmt, double x) {
    if (isnan(x)) return x;
    if (fmt == 0) return (double)(float)x;
    if (x == 0.0 || isinf(x)) return x;
    int mant, emin, sat;
    double maxf;
    if (fmt == 1) { mant = 7; emin = -126; maxf = ldexp(2.0 - ldexp(1.0, -7), 127); sat = 0; }
    else { mant = 3; emin = -6; maxf = 448.0; sat = 1; }
    int e = ilogb(fabs(x));
    if (e < emin) e = emin;
    const int q = e - mant;
    const double r = ldexp(rint(ldexp(x, -q)), q);
    if (fabs(r) > maxf) return sat ? copysign(maxf, x) : copysign(INFINITY, x);
    return r;
}

static double max_finite_of(int fmt) {
    if (fmt == 1) return ldexp(2.0 - ldexp(1.0, -7), 127);
    if (fmt == 2) return 448.0;
    return 3.4028234663852886e38;
}

static int64_t block_of(int gran, int64_t r, int64_t c, int64_t cols, int64_t gs) {
    switch (gran) {
        case 0: return 0;
        case 1: return r;
        case 2: return c;
        default: return r * ((cols + gs - 1) / gs) + c / gs;
    }
}

/* numerics.cpp:88-160: block absmax; scale = absmax / max_finite (1 for an
 * all-zero block); codes = round_to(fmt, x / scale). */
int orc_quantize(const double* x, int64_t rows, int64_t cols, int gran, int64_t group_size,
                 int fmt, double* codes, double* scales, int64_t* num_blocks) {
    if (rows < 0 || cols < 0) return -2;
    if (gran == 3 && group_size < 1) return -2;
    int64_t nb = 1;
    if (gran == 1) nb = rows;
    else if (gran == 2) nb = cols;
    else if (gran == 3) nb = rows * ((cols + group_size - 1) / group_size);
    if (nb < 1) nb = 1;
    for (int64_t b = 0; b < nb; ++b) scales[b] = 0.0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            const double v = fabs(x[r * cols + c]);
            double* m = &scales[block_of(gran, r, c, cols, group_size)];
            if (v > *m) *m = v;
        }
    const double mf = max_finite_of(fmt);
    for (int64_t b = 0; b < nb; ++b) scales[b] = scales[b] > 0.0 ? scales[b] / mf : 1.0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            codes[r * cols + c] =
                orc_round_to(fmt, x[r * cols + c] / scales[block_of(gran, r, c, cols, group_size)]);
    *num_blocks = nb;
    return 0;
}

/* numerics.cpp:172-192. */
int orc_emulate_reduce(const double* v, int64_t ranks, int64_t dim, int kind, double* out) {
    if (ranks < 2) return -2;
    for (int64_t i = 0; i < dim; ++i) {
        double acc = orc_round_to(1, v[i]);
        for (int64_t r = 1; r < ranks; ++r) {
            acc += orc_round_to(1, v[r * dim + i]);
            if (kind == 0 && r + 1 < ranks) acc = orc_round_to(1, acc);
        }
        out[i] = acc;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* dense fp32 path (parity unpinned; conventions pinned, see header)   */
/* ------------------------------------------------------------------ */

static inline double silu_d(double v) { return v / (1.0 + exp(-v)); }
static inline double dsilu_d(double v) {
    const double s = 1.0 / (1.0 + exp(-v));
    return s * (1.0 + v * (1.0 - s));
}

static double dot_f(const float* a, const float* b, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
    return acc;
}

void orc_router_topk(const float* x, const float* wr, int64_t T, int64_t h, int64_t E,
                     int64_t k, float* logits, int32_t* experts, float* gates) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        float* lg = logits + t * E;
        for (int64_t e = 0; e < E; ++e) lg[e] = (float)dot_f(x + t * h, wr + e * h, h);
        /* selection: largest first, ties -> lower expert id */
        for (int64_t j = 0; j < k; ++j) {
            int32_t best = -1;
            for (int64_t e = 0; e < E; ++e) {
                int taken = 0;
                for (int64_t i = 0; i < j; ++i) taken |= experts[t * k + i] == e;
                if (taken) continue;
                if (best < 0 || lg[e] > lg[best]) best = (int32_t)e;
            }
            experts[t * k + j] = best;
        }
        double m = lg[experts[t * k]], s = 0.0;
        for (int64_t j = 0; j < k; ++j) s += exp((double)lg[experts[t * k + j]] - m);
        for (int64_t j = 0; j < k; ++j)
            gates[t * k + j] = (float)(exp((double)lg[experts[t * k + j]] - m) / s);
    }
}

/* One (token, slot) through the expert: fc1 -> SwiGLU (-> gate) -> fc2
 * (graph.cpp:288-296). Writes fc1 (2f) and fc2_in (f) scratch and returns
 * fc2_out (h, before the after-fc2 gate). */
static void expert_fwd(const float* xt, const float* w1e, const float* w2e, int64_t h,
                       int64_t f, double g, int gate_after, double* fc1, double* fc2_in,
                       double* out) {
    for (int64_t j = 0; j < 2 * f; ++j) fc1[j] = dot_f(xt, w1e + j * h, h);
    for (int64_t j = 0; j < f; ++j) {
        double v = fc1[j] * silu_d(fc1[f + j]); /* a * silu(b), numerics.cpp:262-268 */
        if (!gate_after) v *= g;
        fc2_in[j] = v;
    }
    for (int64_t i = 0; i < h; ++i) {
        const float* w = w2e + i * f;
        double acc = 0.0;
        for (int64_t j = 0; j < f; ++j) acc += (double)w[j] * fc2_in[j];
        out[i] = acc;
    }
}

void orc_moe_forward(const float* x, const int32_t* experts, const float* gates,
                     const uint8_t* dropped, const float* w1, const float* w2, int64_t h,
                     int64_t f, int64_t k, int gate_after, const int64_t* tokens, int64_t nt,
                     float* y) {
#pragma omp parallel
    {
        double* fc1 = (double*)malloc(sizeof(double) * (size_t)(2 * f));
        double* fc2_in = (double*)malloc(sizeof(double) * (size_t)f);
        double* out = (double*)malloc(sizeof(double) * (size_t)h);
        double* acc = (double*)malloc(sizeof(double) * (size_t)h);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < nt; ++i) {
            const int64_t t = tokens[i];
            for (int64_t c = 0; c < h; ++c) acc[c] = 0.0;
            if (!dropped[t]) {
                for (int64_t j = 0; j < k; ++j) {
                    const int32_t e = experts[t * k + j];
                    const double g = gates[t * k + j];
                    expert_fwd(x + t * h, w1 + (int64_t)e * 2 * f * h, w2 + (int64_t)e * h * f, h,
                               f, g, gate_after, fc1, fc2_in, out);
                    /* combine: fixed slot order, wide accumulation (a2a_fp32
                     * semantics, numerics.cpp:172-192) */
                    for (int64_t c = 0; c < h; ++c) acc[c] += gate_after ? g * out[c] : out[c];
                }
            }
            for (int64_t c = 0; c < h; ++c) y[i * h + c] = (float)acc[c];
        }
        free(fc1); free(fc2_in); free(out); free(acc);
    }
}

void orc_moe_backward(const float* x, const float* dy, const int32_t* experts,
                      const float* gates, const float* logits, const uint8_t* dropped,
                      const float* w1, const float* w2, const float* wr, int64_t h, int64_t f,
                      int64_t E, int64_t k, int gate_after, const int64_t* tokens, int64_t nt,
                      float* dx, float* dgates, float* dw1, float* dw2, float* dwr) {
    /* per (token, slot) intermediates for the weight-gradient pass */
    float* dfc1_all = (float*)calloc((size_t)(nt * k * 2 * f), sizeof(float));
    float* fc2in_all = (float*)calloc((size_t)(nt * k * f), sizeof(float));
    float* dout_all = (float*)calloc((size_t)(nt * k * h), sizeof(float));
    float* dlog_all = (float*)calloc((size_t)(nt * E), sizeof(float));
#pragma omp parallel
    {
        double* fc1 = (double*)malloc(sizeof(double) * (size_t)(2 * f));
        double* fc2_in = (double*)malloc(sizeof(double) * (size_t)f);
        double* out = (double*)malloc(sizeof(double) * (size_t)h);
        double* dfc2 = (double*)malloc(sizeof(double) * (size_t)f);
        double* dxa = (double*)malloc(sizeof(double) * (size_t)h);
        double* dg = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < nt; ++i) {
            const int64_t t = tokens[i];
            for (int64_t c = 0; c < h; ++c) dxa[c] = 0.0;
            for (int64_t j = 0; j < k; ++j) dg[j] = 0.0;
            if (!dropped[t]) {
                for (int64_t j = 0; j < k; ++j) {
                    const int32_t e = experts[t * k + j];
                    const double g = gates[t * k + j];
                    const float* w1e = w1 + (int64_t)e * 2 * f * h;
                    const float* w2e = w2 + (int64_t)e * h * f;
                    expert_fwd(x + t * h, w1e, w2e, h, f, g, gate_after, fc1, fc2_in, out);
                    float* dout = dout_all + (i * k + j) * h;
                    /* d fc2_out */
                    if (gate_after) {
                        double s = 0.0;
                        for (int64_t c = 0; c < h; ++c) {
                            s += (double)dy[t * h + c] * out[c];
                            dout[c] = (float)(g * dy[t * h + c]);
                        }
                        dg[j] += s;
                    } else {
                        for (int64_t c = 0; c < h; ++c) dout[c] = dy[t * h + c];
                    }
                    /* d fc2_in = W2^T d fc2_out */
                    for (int64_t q = 0; q < f; ++q) dfc2[q] = 0.0;
                    for (int64_t c = 0; c < h; ++c) {
                        const double d = dout[c];
                        const float* w = w2e + c * f;
                        for (int64_t q = 0; q < f; ++q) dfc2[q] += d * (double)w[q];
                    }
                    float* dfc1 = dfc1_all + (i * k + j) * 2 * f;
                    const double gg = gate_after ? 1.0 : g;
                    double sg = 0.0;
                    for (int64_t q = 0; q < f; ++q) {
                        const double a = fc1[q], b = fc1[f + q];
                        sg += dfc2[q] * a * silu_d(b);
                        dfc1[q] = (float)(dfc2[q] * gg * silu_d(b));
                        dfc1[f + q] = (float)(dfc2[q] * gg * a * dsilu_d(b));
                        fc2in_all[(i * k + j) * f + q] = (float)fc2_in[q];
                    }
                    if (!gate_after) dg[j] += sg;
                    /* dx += W1e^T dfc1, row by row (contiguous in W1e) */
                    for (int64_t q = 0; q < 2 * f; ++q) {
                        const double d = dfc1[q];
                        const float* w = w1e + q * h;
                        for (int64_t c = 0; c < h; ++c) dxa[c] += d * (double)w[c];
                    }
                }
                /* router: gates = softmax over selected logits */
                double sdg = 0.0;
                for (int64_t j = 0; j < k; ++j) sdg += gates[t * k + j] * dg[j];
                float* dl = dlog_all + i * E;
                for (int64_t j = 0; j < k; ++j)
                    dl[experts[t * k + j]] = (float)(gates[t * k + j] * (dg[j] - sdg));
                for (int64_t c = 0; c < h; ++c) {
                    double acc = 0.0;
                    for (int64_t e = 0; e < E; ++e) acc += (double)dl[e] * (double)wr[e * h + c];
                    dxa[c] += acc;
                }
            }
            for (int64_t c = 0; c < h; ++c) dx[i * h + c] = (float)dxa[c];
            for (int64_t j = 0; j < k; ++j) dgates[i * k + j] = (float)dg[j];
        }
        free(fc1); free(fc2_in); free(out); free(dfc2); free(dxa); free(dg);
    }
    (void)logits;
    if (dw1 || dw2) {
        /* weight gradients: parallel over output rows, tokens in order */
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t row = 0; row < E * 2 * f; ++row) {
            const int64_t e = row / (2 * f), q = row % (2 * f);
            if (!dw1) continue;
            float* dst = dw1 + row * h;
            for (int64_t i = 0; i < nt; ++i) {
                const int64_t t = tokens[i];
                if (dropped[t]) continue;
                for (int64_t j = 0; j < k; ++j) {
                    if (experts[t * k + j] != e) continue;
                    const float d = dfc1_all[(i * k + j) * 2 * f + q];
                    for (int64_t c = 0; c < h; ++c) dst[c] += d * x[t * h + c];
                }
            }
        }
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t row = 0; row < E * h; ++row) {
            const int64_t e = row / h, c = row % h;
            if (!dw2) continue;
            float* dst = dw2 + row * f;
            for (int64_t i = 0; i < nt; ++i) {
                const int64_t t = tokens[i];
                if (dropped[t]) continue;
                for (int64_t j = 0; j < k; ++j) {
                    if (experts[t * k + j] != e) continue;
                    const float d = dout_all[(i * k + j) * h + c];
                    const float* src = fc2in_all + (i * k + j) * f;
                    for (int64_t q = 0; q < f; ++q) dst[q] += d * src[q];
                }
            }
        }
    }
    if (dwr) {
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < E; ++e)
            for (int64_t i = 0; i < nt; ++i) {
                const float d = dlog_all[i * E + e];
                if (d == 0.0f) continue;
                const int64_t t = tokens[i];
                for (int64_t c = 0; c < h; ++c) dwr[e * h + c] += d * x[t * h + c];
            }
    }
    free(dfc1_all); free(fc2in_all); free(dout_all); free(dlog_all);
}

/* ------------------------------------------------------------------ */
/* bf16-input restatement for full-shape sampled parity                 */
/* ------------------------------------------------------------------ */
/* The same math as orc_moe_forward / orc_moe_backward above, reading the
 * bf16 tensors the GPU holds (uint16 bit patterns widened exactly to fp32)
 * so full-size weights (DeepSeek shape: 22 GB of bf16) need not be widened
 * on the host. Accumulation in binary64, rows contiguous in the weights. */

static inline double bf2d(uint16_t u) {
    union { uint32_t u; float f; } v;
    v.u = (uint32_t)u << 16;
    return (double)v.f;
}

static double dot_bd(const double* a, const uint16_t* b, int64_t n) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 += a[i] * bf2d(b[i]);
        s1 += a[i + 1] * bf2d(b[i + 1]);
        s2 += a[i + 2] * bf2d(b[i + 2]);
        s3 += a[i + 3] * bf2d(b[i + 3]);
    }
    for (; i < n; ++i) s0 += a[i] * bf2d(b[i]);
    return (s0 + s1) + (s2 + s3);
}

/* y, dx and dgates of the sampled tokens (graph.cpp:288-296 forward,
 * :333-401 backward; gates = softmax over the selected logits, so the
 * router term of dx is W_r^T dlogits with dlogits_e = g_e (dg_e - sum g dg)).
 * x[T,h], dy[T,h] (may be NULL: forward only), w1[E,2f,h] ([a|b] rows),
 * w2[E,h,f], wr[E,h] (may be NULL: no router term) are bf16 bit patterns.
 * Outputs y[nt,h], dx[nt,h], dgates[nt,k] (dx/dgates ignored when dy NULL). */
void orc_moe_rows_bf16(const uint16_t* x, const uint16_t* dy, const int32_t* experts,
                       const float* gates, const uint8_t* dropped, const uint16_t* w1,
                       const uint16_t* w2, const uint16_t* wr, int64_t h, int64_t f, int64_t E,
                       int64_t k, int gate_after, const int64_t* tokens, int64_t nt, float* y,
                       float* dx, float* dgates) {
#pragma omp parallel
    {
        double* xt = (double*)malloc(sizeof(double) * (size_t)h);
        double* dyt = (double*)malloc(sizeof(double) * (size_t)h);
        double* fc1 = (double*)malloc(sizeof(double) * (size_t)(2 * f));
        double* fc2_in = (double*)malloc(sizeof(double) * (size_t)f);
        double* out = (double*)malloc(sizeof(double) * (size_t)h);
        double* dout = (double*)malloc(sizeof(double) * (size_t)h);
        double* dfc2 = (double*)malloc(sizeof(double) * (size_t)f);
        double* dfc1 = (double*)malloc(sizeof(double) * (size_t)(2 * f));
        double* ya = (double*)malloc(sizeof(double) * (size_t)h);
        double* dxa = (double*)malloc(sizeof(double) * (size_t)h);
        double dg[64];
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < nt; ++i) {
            const int64_t t = tokens[i];
            for (int64_t c = 0; c < h; ++c) {
                xt[c] = bf2d(x[t * h + c]);
                dyt[c] = dy ? bf2d(dy[t * h + c]) : 0.0;
                ya[c] = 0.0;
                dxa[c] = 0.0;
            }
            for (int64_t j = 0; j < k; ++j) dg[j] = 0.0;
            if (!dropped[t]) {
                for (int64_t j = 0; j < k; ++j) {
                    const int32_t e = experts[t * k + j];
                    const double g = gates[t * k + j];
                    const uint16_t* w1e = w1 + (int64_t)e * 2 * f * h;
                    const uint16_t* w2e = w2 + (int64_t)e * h * f;
                    for (int64_t q = 0; q < 2 * f; ++q) fc1[q] = dot_bd(xt, w1e + q * h, h);
                    for (int64_t q = 0; q < f; ++q)
                        fc2_in[q] = fc1[q] * silu_d(fc1[f + q]) * (gate_after ? 1.0 : g);
                    for (int64_t c = 0; c < h; ++c) out[c] = dot_bd(fc2_in, w2e + c * f, f);
                    for (int64_t c = 0; c < h; ++c) ya[c] += gate_after ? g * out[c] : out[c];
                    if (!dy) continue;
                    if (gate_after) {
                        double s = 0.0;
                        for (int64_t c = 0; c < h; ++c) {
                            s += dyt[c] * out[c];
                            dout[c] = g * dyt[c];
                        }
                        dg[j] += s;
                    } else {
                        for (int64_t c = 0; c < h; ++c) dout[c] = dyt[c];
                    }
                    for (int64_t q = 0; q < f; ++q) dfc2[q] = 0.0;
                    for (int64_t c = 0; c < h; ++c) {
                        const double d = dout[c];
                        const uint16_t* w = w2e + c * f;
                        for (int64_t q = 0; q < f; ++q) dfc2[q] += d * bf2d(w[q]);
                    }
                    const double gg = gate_after ? 1.0 : g;
                    double sg = 0.0;
                    for (int64_t q = 0; q < f; ++q) {
                        const double a = fc1[q], b = fc1[f + q];
                        sg += dfc2[q] * a * silu_d(b);
                        dfc1[q] = dfc2[q] * gg * silu_d(b);
                        dfc1[f + q] = dfc2[q] * gg * a * dsilu_d(b);
                    }
                    if (!gate_after) dg[j] += sg;
                    for (int64_t q = 0; q < 2 * f; ++q) {
                        const double d = dfc1[q];
                        const uint16_t* w = w1e + q * h;
                        for (int64_t c = 0; c < h; ++c) dxa[c] += d * bf2d(w[c]);
                    }
                }
                if (dy && wr) {
                    double sdg = 0.0;
                    for (int64_t j = 0; j < k; ++j) sdg += gates[t * k + j] * dg[j];
                    for (int64_t j = 0; j < k; ++j) {
                        const double dl = gates[t * k + j] * (dg[j] - sdg);
                        const uint16_t* w = wr + (int64_t)experts[t * k + j] * h;
                        for (int64_t c = 0; c < h; ++c) dxa[c] += dl * bf2d(w[c]);
                    }
                }
            }
            for (int64_t c = 0; c < h; ++c) y[i * h + c] = (float)ya[c];
            if (dy) {
                for (int64_t c = 0; c < h; ++c) dx[i * h + c] = (float)dxa[c];
                for (int64_t j = 0; j < k; ++j) dgates[i * k + j] = (float)dg[j];
            }
        }
        free(xt); free(dyt); free(fc1); free(fc2_in); free(out); free(dout); free(dfc2);
        free(dfc1); free(ya); free(dxa);
    }
    (void)E;
}

/* Sampled columns of the expert weight gradients over ALL tokens
 * (graph.cpp:376-398 wgrad nodes). For each sampled intermediate column
 * j = cols[c] in [0, f):
 *   dw1_rows[e][2c]   = dW1[e][j, :]     = sum_t dfc1_a[t, j] x[t, :]
 *   dw1_rows[e][2c+1] = dW1[e][f+j, :]   = sum_t dfc1_b[t, j] x[t, :]
 *   dw2_cols[e][c]    = dW2[e][:, j]     = sum_t dout[t, :] fc2_in[t, j]
 * Column j needs only x.w1[j], x.w1[f+j] and dout.w2[:, j] per row, so the
 * cost is O(T k h) per column. Outputs: dw1_rows [E, 2nc, h], dw2_cols
 * [E, nc, h] (fp32). Parallel over experts; rows of an expert in token order. */
void orc_moe_wgrad_cols_bf16(const uint16_t* x, const uint16_t* dy, const int32_t* experts,
                             const float* gates, const uint8_t* dropped, const uint16_t* w1,
                             const uint16_t* w2, int64_t T, int64_t h, int64_t f, int64_t E,
                             int64_t k, int gate_after, const int64_t* cols, int64_t nc,
                             float* dw1_rows, float* dw2_cols) {
#pragma omp parallel
    {
        double* xt = (double*)malloc(sizeof(double) * (size_t)h);
        double* dout = (double*)malloc(sizeof(double) * (size_t)h);
        double* a1 = (double*)calloc((size_t)(2 * nc * h), sizeof(double));
        double* a2 = (double*)calloc((size_t)(nc * h), sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t e = 0; e < E; ++e) {
            memset(a1, 0, sizeof(double) * (size_t)(2 * nc * h));
            memset(a2, 0, sizeof(double) * (size_t)(nc * h));
            const uint16_t* w1e = w1 + e * 2 * f * h;
            const uint16_t* w2e = w2 + e * h * f;
            for (int64_t t = 0; t < T; ++t) {
                if (dropped[t]) continue;
                for (int64_t s = 0; s < k; ++s) {
                    if (experts[t * k + s] != e) continue;
                    const double g = gates[t * k + s];
                    for (int64_t c = 0; c < h; ++c) {
                        xt[c] = bf2d(x[t * h + c]);
                        dout[c] = (gate_after ? g : 1.0) * bf2d(dy[t * h + c]);
                    }
                    const double gg = gate_after ? 1.0 : g;
                    for (int64_t ci = 0; ci < nc; ++ci) {
                        const int64_t j = cols[ci];
                        const double a = dot_bd(xt, w1e + j * h, h);
                        const double b = dot_bd(xt, w1e + (f + j) * h, h);
                        double d2 = 0.0;
                        for (int64_t c = 0; c < h; ++c) d2 += dout[c] * bf2d(w2e[c * f + j]);
                        const double da = d2 * gg * silu_d(b);
                        const double db = d2 * gg * a * dsilu_d(b);
                        const double fin = a * silu_d(b) * gg;
                        double* r1 = a1 + (2 * ci) * h;
                        double* r2 = a1 + (2 * ci + 1) * h;
                        double* r3 = a2 + ci * h;
                        for (int64_t c = 0; c < h; ++c) {
                            r1[c] += da * xt[c];
                            r2[c] += db * xt[c];
                            r3[c] += fin * dout[c];
                        }
                    }
                }
            }
            for (int64_t i = 0; i < 2 * nc * h; ++i) dw1_rows[e * 2 * nc * h + i] = (float)a1[i];
            for (int64_t i = 0; i < nc * h; ++i) dw2_cols[e * nc * h + i] = (float)a2[i];
        }
        free(xt); free(dout); free(a1); free(a2);
    }
}
