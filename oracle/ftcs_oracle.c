/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference's FTCS hot path on the 8^Dims sparse
 * block grid (porediff, /root/reference/proj/include/porediff/solver.hpp):
 *   - gather                solver.hpp:360-383
 *   - process_chunk         solver.hpp:385-455
 *   - step reductions       solver.hpp:250-278
 *   - pairwise_sum          parallel.hpp:68-84
 *   - snapshot_diagnostics  solver.hpp:282-301
 *   - max_diffusivity       solver.hpp:139-154
 *   - stability_dt          solver.hpp:111-120
 *   - validate              solver.hpp:304-331
 *   - build_neighbor_table  solver.hpp:333-351
 *   - run_simulation        solver.hpp:489-519
 * Compiled with -ffp-contract=off like the reference (CMakeLists.txt:14) so
 * every expression rounds exactly as the reference's does.
 *
 * Parity of this restatement is PINNED against the reference itself
 * (oracle/_ref/libporediff_ref.so, built from the unmodified reference
 * headers by oracle/Makefile) and against the committed golden vectors in
 * tests/golden/ (tests/test_oracle.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. It is single-threaded (cores = 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "porediff_b200.h"

#define OCAT_(a, b) a##b
#define OCAT(a, b) OCAT_(a, b)

typedef struct {
    int dims, V, W;
    int64_t size[3];
    double spacing[3];
    double cell_volume;
    int64_t n_chunks;
    const int32_t* keys;
    const uint64_t* masks;
} OracleGrid;

typedef struct {
    const pd_sim_config* cfg;
    int32_t* nbr;
    double *mass, *mn, *mx, *scratch;
    int64_t bad_ordinal, bad_step;
    int bad_offset;
} OracleRun;

static char g_msg[512];
const char* oracle_last_error(void) { return g_msg; }

static inline int oracle_test(const OracleGrid* g, int64_t i, int off) {
    return (int)((g->masks[i * g->W + (off >> 6)] >> (off & 63)) & 1u);
}

/* parallel.hpp:68-84: level-by-level adjacent pairs, odd tail carried. */
double oracle_pairwise_sum(const double* v, int64_t n, double* scratch) {
    if (n == 0) return 0.0;
    memcpy(scratch, v, sizeof(double) * (size_t)n);
    while (n > 1) {
        const int64_t half = n / 2;
        for (int64_t i = 0; i < half; ++i) scratch[i] = scratch[2 * i] + scratch[2 * i + 1];
        if (n % 2 == 1) {
            scratch[half] = scratch[n - 1];
            n = half + 1;
        } else {
            n = half;
        }
    }
    return scratch[0];
}

#define OT double
#define OSFX _f64
#include "ftcs_oracle_body.h"
#undef OT
#undef OSFX
#define OT float
#define OSFX _f32
#include "ftcs_oracle_body.h"
#undef OT
#undef OSFX

/* stability_dt (solver.hpp:111-120) */
double oracle_stability_dt(int dims, const double* spacing, double d_max) {
    double inv_sum = 0.0;
    for (int a = 0; a < dims; ++a) inv_sum += 1.0 / (spacing[a] * spacing[a]);
    return 1.0 / (2.0 * d_max) / inv_sum;
}

/* build_neighbor_table (solver.hpp:333-351) via a dense linear-index table
 * (the reference's table_, sparse_block_grid.hpp:299). */
static int32_t* build_nbr(const OracleGrid* g) {
    int64_t cc[3] = {1, 1, 1}, table = 1;
    for (int a = 0; a < g->dims; ++a) {
        cc[a] = (g->size[a] + 7) / 8;
        table *= cc[a];
    }
    int32_t* tab = (int32_t*)malloc(sizeof(int32_t) * (size_t)table);
    for (int64_t t = 0; t < table; ++t) tab[t] = -1;
    for (int64_t i = 0; i < g->n_chunks; ++i) {
        int64_t lin = 0;
        for (int a = g->dims - 1; a >= 0; --a) lin = lin * cc[a] + g->keys[i * g->dims + a];
        tab[lin] = (int32_t)i;
    }
    int32_t* nbr = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n_chunks * 2 * g->dims + 1));
    for (int64_t i = 0; i < g->n_chunks; ++i)
        for (int a = 0; a < g->dims; ++a)
            for (int s = 0; s < 2; ++s) {
                int64_t k[3];
                for (int b = 0; b < g->dims; ++b) k[b] = g->keys[i * g->dims + b];
                k[a] += s == 0 ? -1 : 1;
                int32_t o = -1;
                if (k[a] >= 0 && k[a] < cc[a]) {
                    int64_t lin = 0;
                    for (int b = g->dims - 1; b >= 0; --b) lin = lin * cc[b] + k[b];
                    o = tab[lin];
                }
                nbr[i * 2 * g->dims + a * 2 + s] = o;
            }
    free(tab);
    return nbr;
}

/* %.17g formatting of format_scalar<double> (scalar_text.hpp:21-28). */
static void fmt17(char* buf, size_t n, double v) {
    if (isnan(v))
        snprintf(buf, n, "nan");
    else
        snprintf(buf, n, "%.*g", 17, v);
}

/* run_simulation (solver.hpp:489-519) on raw chunk arrays.
 * slabs: phi, u, d, u_next, src (src may be NULL) — n_chunks*V scalars of
 * tbytes each. u and u_next are advanced in place; on return *swapped says
 * whether the logical "u" now lives in the u_next buffer (odd step count).
 * factors: per-step T(time_factor(s*dt)) or NULL. rows: >= n/record+2.
 * Returns a PD_E_* code; the message via oracle_last_error(). */
int oracle_run_simulation(int dims, int tbytes, const int64_t* size, const double* spacing,
                          int64_t n_chunks, const int32_t* keys, const uint64_t* masks,
                          const void* phi, void* u, const void* d, void* u_next,
                          const void* src, const pd_sim_config* cfg, const double* factors,
                          pd_diag* rows, int64_t* n_rows, int* swapped) {
    OracleGrid g;
    memset(&g, 0, sizeof g);
    g.dims = dims;
    g.V = dims == 2 ? 64 : 512;
    g.W = g.V / 64;
    g.cell_volume = 1.0;
    for (int a = 0; a < dims; ++a) {
        g.size[a] = size[a];
        g.spacing[a] = spacing[a];
        g.cell_volume *= spacing[a];
    }
    g.n_chunks = n_chunks;
    g.keys = keys;
    g.masks = masks;
    *n_rows = 0;
    *swapped = 0;
    g_msg[0] = 0;

    /* validate (solver.hpp:304-331) */
    if (!(cfg->dt > 0.0) || !isfinite(cfg->dt)) {
        snprintf(g_msg, sizeof g_msg, "time step must be positive and finite");
        return PD_E_INPUT;
    }
    if (cfg->n_steps < 1) {
        snprintf(g_msg, sizeof g_msg, "step count must be at least 1");
        return PD_E_INPUT;
    }
    if (cfg->record_every < 1) {
        snprintf(g_msg, sizeof g_msg, "record_every must be at least 1");
        return PD_E_INPUT;
    }
    if (!(cfg->b_low < cfg->b_up)) {
        snprintf(g_msg, sizeof g_msg, "phase band is empty (b_low must be < b_up)");
        return PD_E_INPUT;
    }
    if (cfg->boundary_epsilon < 0.0 || !isfinite(cfg->boundary_epsilon)) {
        snprintf(g_msg, sizeof g_msg, "boundary_epsilon must be finite and >= 0");
        return PD_E_INPUT;
    }
    if (cfg->reaction_kind == PD_REACTION_SURFACE_SINK) {
        if (cfg->rate < 0.0) {
            snprintf(g_msg, sizeof g_msg, "surface sink rate must be >= 0");
            return PD_E_INPUT;
        }
        if (!(cfg->band_half_width > 0.0)) {
            snprintf(g_msg, sizeof g_msg, "surface sink band half-width must be > 0");
            return PD_E_INPUT;
        }
    }
    if (cfg->reaction_kind == PD_REACTION_VOLUMETRIC && !src) {
        snprintf(g_msg, sizeof g_msg, "unknown property (source channel)");
        return PD_E_PROPERTY;
    }

    OracleRun r;
    memset(&r, 0, sizeof r);
    r.cfg = cfg;
    r.nbr = build_nbr(&g);
    const size_t nc = (size_t)(n_chunks > 0 ? n_chunks : 1);
    r.mass = (double*)malloc(sizeof(double) * nc);
    r.mn = (double*)malloc(sizeof(double) * nc);
    r.mx = (double*)malloc(sizeof(double) * nc);
    r.scratch = (double*)malloc(sizeof(double) * nc);
    r.bad_ordinal = -1;
    int rc = PD_OK;

    /* stability gate (solver.hpp:495-503, bound from solver.hpp:220-224) */
    if (cfg->enforce_stability) {
        const double dmax = tbytes == 8 ? max_active_f64(&g, (const double*)d)
                                        : max_active_f32(&g, (const float*)d);
        const double bound = dmax > 0.0 ? oracle_stability_dt(dims, spacing, dmax) : INFINITY;
        if (!(cfg->dt < bound)) {
            char a[64], b[64], c[64];
            fmt17(a, sizeof a, cfg->dt);
            fmt17(b, sizeof b, bound);
            fmt17(c, sizeof c, dmax);
            snprintf(g_msg, sizeof g_msg,
                     "time step %s violates the explicit stability bound %s (dt must be "
                     "strictly below it; max D = %s)",
                     a, b, c);
            rc = PD_E_STABILITY;
            goto done;
        }
    }

    /* step-0 row (solver.hpp:510) */
    if (tbytes == 8)
        snapshot_f64(&g, &r, (const double*)u, &rows[(*n_rows)++]);
    else
        snapshot_f32(&g, &r, (const float*)u, &rows[(*n_rows)++]);

    {
        void* cur = u;
        void* nxt = u_next;
        for (int64_t s = 0; s < cfg->n_steps; ++s) {
            pd_diag row;
            const double f = factors ? factors[s] : 1.0;
            if (tbytes == 8)
                rc = step_f64(&g, &r, (const double*)phi, (const double*)cur,
                              (const double*)d, (const double*)src, (double*)nxt,
                              (double)f, s, &row);
            else
                rc = step_f32(&g, &r, (const float*)phi, (const float*)cur, (const float*)d,
                              (const float*)src, (float*)nxt, (float)f, s, &row);
            if (rc != PD_OK) {
                int len = snprintf(g_msg, sizeof g_msg, "non-finite value at step %lld, node (",
                                   (long long)r.bad_step);
                for (int a = 0; a < dims; ++a) {
                    const int64_t idx = ((int64_t)keys[r.bad_ordinal * dims + a] << 3) |
                                        ((r.bad_offset >> (3 * a)) & 7);
                    len += snprintf(g_msg + len, sizeof g_msg - (size_t)len, "%s%lld",
                                    a ? "," : "", (long long)idx);
                }
                snprintf(g_msg + len, sizeof g_msg - (size_t)len, ")");
                goto done;
            }
            /* swap_channels (solver.hpp:262) */
            void* t = cur;
            cur = nxt;
            nxt = t;
            *swapped = !*swapped;
            if (!isfinite(row.total_mass)) {
                snprintf(g_msg, sizeof g_msg, "non-finite total mass at step %lld",
                         (long long)(s + 1));
                rc = PD_E_NUMERIC;
                goto done;
            }
            if ((s + 1) % cfg->record_every == 0 || s + 1 == cfg->n_steps)
                rows[(*n_rows)++] = row;
        }
    }
done:
    free(r.nbr);
    free(r.mass);
    free(r.mn);
    free(r.mx);
    free(r.scratch);
    return rc;
}

/* total_mass / max_diffusivity on raw arrays (solver.hpp:139-171). */
double oracle_total_mass(int dims, int tbytes, const double* spacing, int64_t n_chunks,
                         const uint64_t* masks, const void* u) {
    OracleGrid g;
    memset(&g, 0, sizeof g);
    g.dims = dims;
    g.V = dims == 2 ? 64 : 512;
    g.W = g.V / 64;
    g.cell_volume = 1.0;
    for (int a = 0; a < dims; ++a) g.cell_volume *= spacing[a];
    g.n_chunks = n_chunks;
    g.masks = masks;
    OracleRun r;
    memset(&r, 0, sizeof r);
    const size_t nc = (size_t)(n_chunks > 0 ? n_chunks : 1);
    r.mass = (double*)malloc(sizeof(double) * nc);
    r.scratch = (double*)malloc(sizeof(double) * nc);
    pd_diag row;
    if (tbytes == 8)
        snapshot_f64(&g, &r, (const double*)u, &row);
    else
        snapshot_f32(&g, &r, (const float*)u, &row);
    free(r.mass);
    free(r.scratch);
    return row.total_mass;
}

/* config.hpp:558-564 */
double oracle_hash_unit_value(uint64_t seed, uint64_t key) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (key + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-53;
}
