/* TEST INFRASTRUCTURE ONLY. Type-generic body of the plain-C restatement of
 * the reference FTCS step; included twice by ftcs_oracle.c with
 * OT = double / float and OSFX = _f64 / _f32. See ftcs_oracle.c. */

/* FtcsStepper::gather (solver.hpp:360-383): face value (u, d) across one face
 * of node `off` (chunk ordinal i) along `axis`, side 0 = low, 1 = high. */
static void OCAT(gather, OSFX)(const OracleGrid* g, const OracleRun* r, int64_t i, int off,
                               int axis, int side, int64_t global, const OT* phi,
                               const OT* u, const OT* d, OT u_c, OT d_c, OT wall,
                               const OT* bcv, OT* fu, OT* fd) {
    const int64_t gg = global + (side == 0 ? -1 : 1);
    const int V = g->V;
    if (gg < 0 || gg >= g->size[axis]) {
        if (r->cfg->bc_type[axis * 2 + side] == PD_BC_DIRICHLET) {
            *fu = bcv[axis * 2 + side];
            *fd = d_c;
        } else {
            *fu = u_c;
            *fd = d_c;
        }
        return;
    }
    const int stride = 1 << (3 * axis);
    const int coord = (off >> (3 * axis)) & 7;
    const int crosses = side == 0 ? coord == 0 : coord == 7;
    int64_t j = i;
    int o2;
    if (!crosses) {
        o2 = side == 0 ? off - stride : off + stride;
    } else {
        j = r->nbr[i * 2 * g->dims + axis * 2 + side];
        o2 = side == 0 ? off + 7 * stride : off - 7 * stride;
        if (j < 0) {
            *fu = u_c;
            *fd = d_c;
            return;
        }
    }
    if (!oracle_test(g, j, o2) || phi[j * V + o2] <= wall) {
        *fu = u_c;
        *fd = d_c;
        return;
    }
    *fu = u[j * V + o2];
    *fd = d[j * V + o2];
}

/* FtcsStepper::process_chunk (solver.hpp:385-455) over every chunk, then the
 * step() reductions (solver.hpp:250-278). Returns 0, or PD_E_NUMERIC with
 * r->bad_* filled for the lowest ordinal / first offset. */
static int OCAT(step, OSFX)(const OracleGrid* g, OracleRun* r, const OT* phi, const OT* u,
                            const OT* d, const OT* src, OT* out, OT source_factor,
                            int64_t step_index, pd_diag* row) {
    const int V = g->V, D = g->dims;
    const pd_sim_config* c = r->cfg;
    OT inv_dx2[3];
    for (int a = 0; a < D; ++a) inv_dx2[a] = (OT)1 / (OT)(g->spacing[a] * g->spacing[a]);
    const OT dt = (OT)c->dt;
    const OT wall = (OT)c->b_low + (OT)c->boundary_epsilon;
    double hmin = g->spacing[0];
    for (int a = 1; a < D; ++a) hmin = hmin < g->spacing[a] ? hmin : g->spacing[a];
    const double sink_band = c->band_half_width * hmin;
    const OT neg_k = -(OT)c->rate;
    OT bcv[6];
    for (int f = 0; f < 6; ++f) bcv[f] = (OT)c->bc_value[f];

    for (int64_t i = 0; i < g->n_chunks; ++i) {
        double mass = 0.0, mn = INFINITY, mx = -INFINITY;
        int bad = -1;
        for (int off = 0; off < V; ++off) {
            if (!oracle_test(g, i, off)) continue;
            const OT u_c = u[i * V + off];
            const OT phi_c = phi[i * V + off];
            OT un;
            if (phi_c <= wall) {
                un = u_c;
            } else {
                const OT d_c = d[i * V + off];
                OT lap = 0;
                for (int a = 0; a < D; ++a) {
                    const int64_t global =
                        ((int64_t)g->keys[i * D + a] << 3) + ((off >> (3 * a)) & 7);
                    OT mu, md, pu, pdv;
                    OCAT(gather, OSFX)(g, r, i, off, a, 0, global, phi, u, d, u_c, d_c, wall,
                                       bcv, &mu, &md);
                    OCAT(gather, OSFX)(g, r, i, off, a, 1, global, phi, u, d, u_c, d_c, wall,
                                       bcv, &pu, &pdv);
                    const OT dh_m = (d_c + md) * (OT)0.5;
                    const OT dh_p = (d_c + pdv) * (OT)0.5;
                    lap += (dh_p * (pu - u_c) - dh_m * (u_c - mu)) * inv_dx2[a];
                }
                OT rate = 0;
                if (c->reaction_kind == PD_REACTION_SURFACE_SINK) {
                    if (fabs((double)phi_c) <= sink_band) rate = neg_k * u_c;
                } else if (c->reaction_kind == PD_REACTION_VOLUMETRIC) {
                    rate = src[i * V + off] * source_factor;
                }
                un = u_c + dt * lap + dt * rate;
            }
            if (!isfinite((double)un) && bad < 0) bad = off;
            out[i * V + off] = un;
            mass += (double)un;
            /* std::min / std::max fold (solver.hpp:447-448) */
            mn = ((double)un < mn) ? (double)un : mn;
            mx = (mx < (double)un) ? (double)un : mx;
        }
        r->mass[i] = mass;
        r->mn[i] = mn;
        r->mx[i] = mx;
        if (bad >= 0 && r->bad_ordinal < 0) {
            r->bad_ordinal = i;
            r->bad_offset = bad;
        }
    }
    if (r->bad_ordinal >= 0) {
        r->bad_step = step_index + 1;
        return PD_E_NUMERIC;
    }
    row->step = step_index + 1;
    row->time = (double)(step_index + 1) * c->dt;
    row->total_mass = oracle_pairwise_sum(r->mass, g->n_chunks, r->scratch) * g->cell_volume;
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < g->n_chunks; ++i) {
        mn = (r->mn[i] < mn) ? r->mn[i] : mn;
        mx = (mx < r->mx[i]) ? r->mx[i] : mx;
    }
    row->min_u = mn;
    row->max_u = mx;
    return PD_OK;
}

/* snapshot_diagnostics (solver.hpp:282-301) / total_mass (solver.hpp:158-171). */
static void OCAT(snapshot, OSFX)(const OracleGrid* g, OracleRun* r, const OT* u, pd_diag* row) {
    const int V = g->V;
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < g->n_chunks; ++i) {
        double s = 0.0;
        for (int off = 0; off < V; ++off)
            if (oracle_test(g, i, off)) {
                const double v = (double)u[i * V + off];
                s += v;
                mn = (v < mn) ? v : mn;
                mx = (mx < v) ? v : mx;
            }
        r->mass[i] = s;
    }
    row->step = 0;
    row->time = 0.0;
    row->total_mass = oracle_pairwise_sum(r->mass, g->n_chunks, r->scratch) * g->cell_volume;
    row->min_u = mn;
    row->max_u = mx;
}

/* max_diffusivity (solver.hpp:139-154). */
static double OCAT(max_active, OSFX)(const OracleGrid* g, const OT* d) {
    double m = -INFINITY;
    int any = 0;
    for (int64_t i = 0; i < g->n_chunks; ++i)
        for (int off = 0; off < g->V; ++off)
            if (oracle_test(g, i, off)) {
                const double v = (double)d[i * g->V + off];
                m = (m < v) ? v : m;
                any = 1;
            }
    return any ? m : 0.0;
}
