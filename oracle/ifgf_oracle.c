/*
 * TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
 *
 * Plain-C restatement of the reference's CF-operator apply (the hot path of
 * /root/reference/proj), used by tests/ as an independent CPU oracle. It consumes the
 * reference's own plan objects (octree boxes, relations, relevant cone segments, proximity
 * pairs, beta tables — exported through oracle/ref_driver.cpp) and recomputes the apply:
 *
 *   level-D fill          ifgf.cpp:312-391   (oracle_level_d_fill)
 *   block transform       ifgf.cpp:92-130    (transform3)
 *   3-D Clenshaw          ifgf.cpp:70-89     (eval3)
 *   cousin evaluation     ifgf.cpp:396-450   (cousin_level)
 *   parent fill           ifgf.cpp:452-568   (parent_level)
 *   ifgf_apply            ifgf.cpp:577-608   (oracle_ifgf_apply, Morton order in/out)
 *   near field            solver.cpp:100-144 (oracle_near_field)
 *   density coefficients  rp.cpp:400-417, chebyshev.cpp:28-61 (oracle_rp_apply)
 *   singular apply        rp.cpp:421-451     (oracle_rp_apply)
 *   cone maps             kernels.cpp:27-48  (to_cone / from_cone)
 *   segment_of            ifgf.cpp:161-176
 *
 * Compiled by oracle/Makefile with -O2 -ffp-contract=off (no FMA), so the segment
 * decisions are the reference's own (same glibc acos/atan2).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

static const double PI = 3.141592653589793;
static const double TWO_PI = 2.0 * 3.141592653589793;
static const double INV4PI = 1.0 / (4.0 * 3.141592653589793);
static const double CONE_ETA = 0.5773502691896258;
static const double HALF_DIAG = 0.8660254037844386;

typedef struct {
    int n, depth;
    double k;
    double root_min[3];
    double root_side;
    const double *px, *py, *pz, *nx, *ny, *nz; /* Morton order */
    /* per level (index d-1) */
    const int* nboxes;
    const int32_t* const* cell;     /* 3 * nb */
    const uint32_t* const* beg;
    const uint32_t* const* end;
    const int32_t* const* child;    /* 8 * nb */
    const int32_t* const* cz_ptr;   /* nb + 1 */
    const int32_t* const* cz_idx;
    const int* ns;
    const int* nc;
    const int* nseg;
    const int32_t* const* seg_box;
    const int32_t* const* seg_gamma;
    const int* npipes;              /* pipes carried at each level */
    const int* pipes;               /* 3 per level: factor codes 1..4 */
    int ps, pang;
} oracle_ifgf;

/* ------------------------------------------------------------ geometry helpers */
static double side_of(const oracle_ifgf* o, int d) { return o->root_side / (double)(1u << (d - 1)); }

static void center_of(const oracle_ifgf* o, int d, int b, double c[3]) {
    const double H = side_of(o, d);
    const int32_t* cl = o->cell[d - 1] + 3 * b;
    for (int a = 0; a < 3; ++a) c[a] = o->root_min[a] + (cl[a] + 0.5) * H;
}

typedef struct {
    double s, th, ph;
} cone_t;

static cone_t to_cone(const double x[3], const double c[3], double h) { /* kernels.cpp:34-48 */
    const double vx = x[0] - c[0], vy = x[1] - c[1], vz = x[2] - c[2];
    const double r = sqrt(vx * vx + vy * vy + vz * vz);
    cone_t o;
    o.s = h / r;
    double ct = vz / r;
    ct = ct > 1.0 ? 1.0 : (ct < -1.0 ? -1.0 : ct);
    o.th = acos(ct);
    double ph = atan2(vy, vx);
    if (ph < 0.0) ph += TWO_PI;
    if (ph >= TWO_PI) ph = 0.0;
    o.ph = ph;
    return o;
}

static void from_cone(double s, double th, double ph, const double c[3], double h, double x[3]) {
    const double r = h / s; /* kernels.cpp:27-32 */
    const double st = sin(th), ct = cos(th);
    x[0] = c[0] + r * st * cos(ph);
    x[1] = c[1] + r * st * sin(ph);
    x[2] = c[2] + r * ct;
}

typedef struct {
    int ns, nc, ps, pang;
    double ds, dth, dph;
    double *sn, *tn, *pn; /* node tables */
} cones_t;

static void cheb_nodes(int n, double* x) {
    for (int k = 0; k < n; ++k) x[k] = cos((2.0 * k + 1.0) * PI / (2.0 * n));
}

static void make_cones(const oracle_ifgf* o, int d, cones_t* L) { /* ifgf.cpp:27-55 */
    L->ns = o->ns[d - 1];
    L->nc = o->nc[d - 1];
    L->ps = o->ps;
    L->pang = o->pang;
    L->ds = CONE_ETA / L->ns;
    L->dth = PI / L->nc;
    L->dph = PI / L->nc;
    double xs[12], xa[12];
    cheb_nodes(L->ps, xs);
    cheb_nodes(L->pang, xa);
    L->sn = malloc(sizeof(double) * L->ns * L->ps);
    L->tn = malloc(sizeof(double) * L->nc * L->pang);
    L->pn = malloc(sizeof(double) * 2 * L->nc * L->pang);
    for (int g = 0; g < L->ns; ++g)
        for (int i = 0; i < L->ps; ++i) L->sn[g * L->ps + i] = g * L->ds + (xs[i] + 1.0) * 0.5 * L->ds;
    for (int g = 0; g < L->nc; ++g)
        for (int i = 0; i < L->pang; ++i) L->tn[g * L->pang + i] = g * L->dth + (xa[i] + 1.0) * 0.5 * L->dth;
    for (int g = 0; g < 2 * L->nc; ++g)
        for (int i = 0; i < L->pang; ++i) L->pn[g * L->pang + i] = g * L->dph + (xa[i] + 1.0) * 0.5 * L->dph;
}

static void free_cones(cones_t* L) {
    free(L->sn);
    free(L->tn);
    free(L->pn);
}

static int segment_of(const cones_t* L, cone_t c, int* g1, int* g2, int* g3) { /* ifgf.cpp:161-176 */
    if (c.s > CONE_ETA + 1e-12) return -1;
    *g1 = (int)floor(c.s / L->ds) + 1;
    if (*g1 > L->ns) *g1 = L->ns;
    if (*g1 < 1) *g1 = 1;
    if (c.th >= PI) {
        *g2 = L->nc;
        *g3 = 2 * L->nc;
        return 0;
    }
    *g2 = (int)floor(c.th / L->dth) + 1;
    if (*g2 > L->nc) *g2 = L->nc;
    if (*g2 < 1) *g2 = 1;
    *g3 = (int)floor(c.ph / L->dph) + 1;
    if (*g3 > 2 * L->nc) *g3 = 2 * L->nc;
    if (*g3 < 1) *g3 = 1;
    return 0;
}

/* relevant segment ordinal of (box, gamma), -1 if absent */
static int seg_lookup(const oracle_ifgf* o, int d, int box, int gamma) {
    const int32_t* sb = o->seg_box[d - 1];
    const int32_t* sg = o->seg_gamma[d - 1];
    int lo = 0, hi = o->nseg[d - 1];
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (sb[mid] < box || (sb[mid] == box && sg[mid] < gamma)) lo = mid + 1;
        else hi = mid;
    }
    return (lo < o->nseg[d - 1] && sb[lo] == box && sg[lo] == gamma) ? lo : -1;
}

/* ------------------------------------------------------------ Chebyshev pieces */
static void transform_matrix(int n, double* M) { /* chebyshev.cpp:169-179 */
    double x[12], t[12];
    cheb_nodes(n, x);
    for (int k = 0; k < n; ++k) {
        t[0] = 1.0;
        if (n > 1) t[1] = x[k];
        for (int i = 2; i < n; ++i) t[i] = 2.0 * x[k] * t[i - 1] - t[i - 2];
        for (int i = 0; i < n; ++i) M[i * n + k] = (i == 0 ? 1.0 : 2.0) / n * t[i];
    }
}

static cplx clenshaw(const cplx* a, int n, double x) { /* ifgf.cpp:70-79 */
    cplx b1 = 0, b2 = 0;
    for (int i = n - 1; i >= 1; --i) {
        const cplx b0 = a[i] + 2.0 * x * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return a[0] + x * b1 - b2;
}

static cplx eval3(const cplx* a, int ps, int pang, double xs, double xt, double xp) { /* ifgf.cpp:81-89 */
    cplx tp[144], pv[12];
    for (int p = 0; p < pang; ++p)
        for (int t = 0; t < pang; ++t) tp[p * pang + t] = clenshaw(a + (p * pang + t) * ps, ps, xs);
    for (int p = 0; p < pang; ++p) pv[p] = clenshaw(tp + p * pang, pang, xt);
    return clenshaw(pv, pang, xp);
}

static void transform3(cplx* a, int ps, int pang, const double* ms, const double* ma) { /* ifgf.cpp:92-130 */
    cplx tmp[12];
    for (int p = 0; p < pang; ++p)
        for (int t = 0; t < pang; ++t) {
            cplx* line = a + (p * pang + t) * ps;
            for (int i = 0; i < ps; ++i) {
                cplx acc = 0;
                for (int k = 0; k < ps; ++k) acc += ms[i * ps + k] * line[k];
                tmp[i] = acc;
            }
            memcpy(line, tmp, sizeof(cplx) * ps);
        }
    for (int p = 0; p < pang; ++p)
        for (int i = 0; i < ps; ++i) {
            cplx* base = a + p * pang * ps + i;
            for (int t = 0; t < pang; ++t) {
                cplx acc = 0;
                for (int k = 0; k < pang; ++k) acc += ma[t * pang + k] * base[k * ps];
                tmp[t] = acc;
            }
            for (int t = 0; t < pang; ++t) base[t * ps] = tmp[t];
        }
    const int stride = pang * ps;
    for (int t = 0; t < pang; ++t)
        for (int i = 0; i < ps; ++i) {
            cplx* base = a + t * ps + i;
            for (int p = 0; p < pang; ++p) {
                cplx acc = 0;
                for (int k = 0; k < pang; ++k) acc += ma[p * pang + k] * base[k * stride];
                tmp[p] = acc;
            }
            for (int p = 0; p < pang; ++p) base[p * stride] = tmp[p];
        }
}

static cplx polar(double r, double th) { return r * cos(th) + I * (r * sin(th)); }

/* ------------------------------------------------------------ IFGF */
static int find_pipe(const int* pipes, int np, int f) {
    for (int i = 0; i < np; ++i)
        if (pipes[i] == f) return i;
    return -1;
}

int oracle_level_d_fill(const oracle_ifgf* o, const double* a_perm_in, double* blocks_out) {
    const int d = o->depth;
    if (d < 3) return 0;
    const cplx* a_perm = (const cplx*)a_perm_in;
    cplx* blocks = (cplx*)blocks_out;
    cones_t L;
    make_cones(o, d, &L);
    const int P = L.ps * L.pang * L.pang;
    const int np = o->npipes[d - 1];
    const int* pipes = o->pipes + 3 * (d - 1);
    double ms[144], ma[144];
    transform_matrix(L.ps, ms);
    transform_matrix(L.pang, ma);
    const double h = HALF_DIAG * side_of(o, d);
    const double k = o->k;
#pragma omp parallel for schedule(dynamic, 8)
    for (int so = 0; so < o->nseg[d - 1]; ++so) {
        const int box = o->seg_box[d - 1][so], gam = o->seg_gamma[d - 1][so];
        const int g1 = gam % L.ns + 1, g2 = (gam / L.ns) % L.nc + 1, g3 = gam / L.ns / L.nc + 1;
        double c[3];
        center_of(o, d, box, c);
        const uint32_t b0 = o->beg[d - 1][box], b1 = o->end[d - 1][box];
        for (int ip = 0; ip < L.pang; ++ip) {
            const double ph = L.pn[(g3 - 1) * L.pang + ip];
            const double cph = cos(ph), sph = sin(ph);
            for (int it = 0; it < L.pang; ++it) {
                const double th = L.tn[(g2 - 1) * L.pang + it];
                const double cth = cos(th), sth = sin(th);
                const double xh[3] = {sth * cph, sth * sph, cth};
                for (int is = 0; is < L.ps; ++is) {
                    const double s = L.sn[(g1 - 1) * L.ps + is];
                    const double soh = s / h, khos = k * h / s;
                    cplx acc[4] = {0, 0, 0, 0};
                    for (uint32_t t = b0; t < b1; ++t) {
                        const double vx = xh[0] - (o->px[t] - c[0]) * soh;
                        const double vy = xh[1] - (o->py[t] - c[1]) * soh;
                        const double vz = xh[2] - (o->pz[t] - c[2]) * soh;
                        const double nv2 = vx * vx + vy * vy + vz * vz;
                        const double nv = sqrt(nv2), inv = 1.0 / nv;
                        const double arg = khos * ((nv2 - 1.0) / (nv + 1.0));
                        const cplx pa = a_perm[t] * polar(1.0, arg);
                        const double dn = vx * o->nx[t] + vy * o->ny[t] + vz * o->nz[t];
                        for (int pi = 0; pi < np; ++pi) {
                            switch (pipes[pi]) {
                                case 1: acc[pi] += pa * inv; break;
                                case 2: acc[pi] += pa * (dn * inv * inv * inv); break;
                                case 3: acc[pi] += pa * (dn * inv * inv); break;
                                default: acc[pi] += pa * ((soh * inv) - I * k) * (dn * inv * inv);
                            }
                        }
                    }
                    const int node = is + L.ps * (it + L.pang * ip);
                    for (int pi = 0; pi < np; ++pi) blocks[((size_t)so * np + pi) * P + node] = acc[pi];
                }
            }
        }
        for (int pi = 0; pi < np; ++pi) transform3(blocks + ((size_t)so * np + pi) * P, L.ps, L.pang, ms, ma);
    }
    free_cones(&L);
    return 0;
}

static int cousin_level(const oracle_ifgf* o, int d, const cplx* data, cplx* single, cplx* dbl) {
    cones_t L;
    make_cones(o, d, &L);
    const int P = L.ps * L.pang * L.pang;
    const int np = o->npipes[d - 1];
    const int* pipes = o->pipes + 3 * (d - 1);
    const double h = HALF_DIAG * side_of(o, d), k = o->k;
    int err = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : err)
    for (int tb = 0; tb < o->nboxes[d - 1]; ++tb) {
        for (int j = o->cz_ptr[d - 1][tb]; j < o->cz_ptr[d - 1][tb + 1]; ++j) {
            const int sb = o->cz_idx[d - 1][j];
            double c[3];
            center_of(o, d, sb, c);
            for (uint32_t t = o->beg[d - 1][tb]; t < o->end[d - 1][tb]; ++t) {
                const double x[3] = {o->px[t], o->py[t], o->pz[t]};
                const cone_t cc = to_cone(x, c, h);
                int g1, g2, g3;
                if (segment_of(&L, cc, &g1, &g2, &g3)) {
                    err |= 1;
                    continue;
                }
                const int so = seg_lookup(o, d, sb, (g1 - 1) + L.ns * ((g2 - 1) + L.nc * (g3 - 1)));
                if (so < 0) {
                    err |= 2;
                    continue;
                }
                const double ls = 2.0 * (cc.s - (g1 - 1) * L.ds) / L.ds - 1.0;
                const double lt = 2.0 * (cc.th - (g2 - 1) * L.dth) / L.dth - 1.0;
                const double lp = 2.0 * (cc.ph - (g3 - 1) * L.dph) / L.dph - 1.0;
                const double r = h / cc.s;
                for (int pi = 0; pi < np; ++pi) {
                    const cplx val = eval3(data + ((size_t)so * np + pi) * P, L.ps, L.pang, ls, lt, lp);
                    switch (pipes[pi]) {
                        case 1: single[t] += polar(INV4PI / r, k * r) * val; break;
                        case 4: dbl[t] += polar(INV4PI / r, k * r) * val; break;
                        case 2: dbl[t] += polar(INV4PI / (r * r), k * r) * val; break;
                        default: dbl[t] += (-I * k) * polar(INV4PI / r, k * r) * val;
                    }
                }
            }
        }
    }
    free_cones(&L);
    return err;
}

static int parent_level(const oracle_ifgf* o, int d, const cplx* child, cplx* out) {
    cones_t PL, CL;
    make_cones(o, d - 1, &PL);
    make_cones(o, d, &CL);
    const int P = PL.ps * PL.pang * PL.pang, cP = CL.ps * CL.pang * CL.pang;
    const int np = o->npipes[d - 2], cnp = o->npipes[d - 1];
    const int* pp = o->pipes + 3 * (d - 2);
    const int* cp = o->pipes + 3 * (d - 1);
    const int cw1 = find_pipe(cp, cnp, 1), cw2 = find_pipe(cp, cnp, 2), cw3 = find_pipe(cp, cnp, 3),
              cw4 = find_pipe(cp, cnp, 4);
    double ms[144], ma[144];
    transform_matrix(PL.ps, ms);
    transform_matrix(PL.pang, ma);
    const double hp = HALF_DIAG * side_of(o, d - 1), hc = HALF_DIAG * side_of(o, d), k = o->k;
    memset(out, 0, sizeof(cplx) * (size_t)o->nseg[d - 2] * np * P);
    int err = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : err)
    for (int so = 0; so < o->nseg[d - 2]; ++so) {
        const int pb = o->seg_box[d - 2][so], gam = o->seg_gamma[d - 2][so];
        const int g1 = gam % PL.ns + 1, g2 = (gam / PL.ns) % PL.nc + 1, g3 = gam / PL.ns / PL.nc + 1;
        double pc[3];
        center_of(o, d - 1, pb, pc);
        for (int ip = 0; ip < PL.pang; ++ip)
            for (int it = 0; it < PL.pang; ++it)
                for (int is = 0; is < PL.ps; ++is) {
                    const double s = PL.sn[(g1 - 1) * PL.ps + is];
                    double x[3];
                    from_cone(s, PL.tn[(g2 - 1) * PL.pang + it], PL.pn[(g3 - 1) * PL.pang + ip], pc, hp, x);
                    const double rp = hp / s;
                    const int node = is + PL.ps * (it + PL.pang * ip);
                    for (int slot = 0; slot < 8; ++slot) {
                        const int ch = o->child[d - 2][8 * pb + slot];
                        if (ch < 0) continue;
                        double cc[3];
                        center_of(o, d, ch, cc);
                        const cone_t c = to_cone(x, cc, hc);
                        int h1, h2, h3;
                        if (segment_of(&CL, c, &h1, &h2, &h3)) {
                            err |= 1;
                            continue;
                        }
                        const int cso = seg_lookup(o, d, ch, (h1 - 1) + CL.ns * ((h2 - 1) + CL.nc * (h3 - 1)));
                        if (cso < 0) {
                            err |= 2;
                            continue;
                        }
                        const double ls = 2.0 * (c.s - (h1 - 1) * CL.ds) / CL.ds - 1.0;
                        const double lt = 2.0 * (c.th - (h2 - 1) * CL.dth) / CL.dth - 1.0;
                        const double lp = 2.0 * (c.ph - (h3 - 1) * CL.dph) / CL.dph - 1.0;
                        const double rc = hc / c.s;
                        /* radius_difference, ifgf.cpp:149-153 */
                        const double sx = cc[0] + pc[0] - 2.0 * x[0], sy = cc[1] + pc[1] - 2.0 * x[1],
                                     sz = cc[2] + pc[2] - 2.0 * x[2];
                        const double dr = (sx * (cc[0] - pc[0]) + sy * (cc[1] - pc[1]) + sz * (cc[2] - pc[2])) / (rc + rp);
                        const cplx ratio1 = polar(rp / rc, k * dr);
                        const cplx* blk = child + (size_t)cso * cnp * cP;
                        for (int pi = 0; pi < np; ++pi) {
                            cplx add = 0;
                            switch (pp[pi]) {
                                case 1: add = ratio1 * eval3(blk + cw1 * cP, CL.ps, CL.pang, ls, lt, lp); break;
                                case 4:
                                    if (cw4 >= 0) {
                                        add = ratio1 * eval3(blk + cw4 * cP, CL.ps, CL.pang, ls, lt, lp);
                                    } else {
                                        const cplx i2 = eval3(blk + cw2 * cP, CL.ps, CL.pang, ls, lt, lp);
                                        const cplx i3 = eval3(blk + cw3 * cP, CL.ps, CL.pang, ls, lt, lp);
                                        add = polar(rp / (rc * rc), k * dr) * i2 + (-I * k) * ratio1 * i3;
                                    }
                                    break;
                                case 2:
                                    add = polar((rp * rp) / (rc * rc), k * dr) * eval3(blk + cw2 * cP, CL.ps, CL.pang, ls, lt, lp);
                                    break;
                                default: add = ratio1 * eval3(blk + cw3 * cP, CL.ps, CL.pang, ls, lt, lp);
                            }
                            out[((size_t)so * np + pi) * P + node] += add;
                        }
                    }
                }
        for (int pi = 0; pi < np; ++pi) transform3(out + ((size_t)so * np + pi) * P, PL.ps, PL.pang, ms, ma);
    }
    free_cones(&PL);
    free_cones(&CL);
    return err;
}

/* Morton-ordered a -> Morton-ordered single/dbl (accumulated into zeroed outputs) */
int oracle_ifgf_apply(const oracle_ifgf* o, const double* a_perm, double* single_out, double* dbl_out) {
    cplx* single = (cplx*)single_out;
    cplx* dbl = (cplx*)dbl_out;
    const int D = o->depth;
    if (D < 3) return 0;
    const int P = o->ps * o->pang * o->pang;
    size_t cap = 0;
    for (int d = 3; d <= D; ++d) {
        const size_t need = (size_t)o->nseg[d - 1] * o->npipes[d - 1] * P;
        if (need > cap) cap = need;
    }
    cplx* cur = calloc(cap ? cap : 1, sizeof(cplx));
    cplx* nxt = calloc(cap ? cap : 1, sizeof(cplx));
    int err = oracle_level_d_fill(o, a_perm, (double*)cur);
    for (int d = D; d >= 3 && !err; --d) {
        err |= cousin_level(o, d, cur, single, dbl);
        if (d > 3) {
            err |= parent_level(o, d, cur, nxt);
            cplx* t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    free(cur);
    free(nxt);
    return err;
}

/* ------------------------------------------------------------ near field (solver.cpp:100-144) */
typedef struct {
    int n;
    double k;
    const double *x, *y, *z, *nx, *ny, *nz; /* original order */
    const double* jw;                       /* J w per node */
    const int32_t* patch_of;
    const int32_t* leaf_of;
    const uint32_t* perm;
    const uint32_t *leaf_beg, *leaf_end;
    const int32_t *nb_ptr, *nb_idx;
    const uint32_t* tpb;
    const int32_t* pair_patch;
    const uint32_t *far_begin, *far_end, *far_nodes;
} oracle_near;

static void kernels(const oracle_near* o, int l, int m, cplx* g, cplx* dg) {
    const double dx = o->x[l] - o->x[m], dy = o->y[l] - o->y[m], dz = o->z[l] - o->z[m];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    *g = polar(INV4PI / r, o->k * r); /* kernels.cpp:12-25 */
    const double dn = dx * o->nx[m] + dy * o->ny[m] + dz * o->nz[m];
    *dg = polar(1.0, o->k * r) * (1.0 - I * (o->k * r)) * (dn * INV4PI / (r * r * r));
}

int oracle_near_field(const oracle_near* o, const double* phi_in, double* S_out, double* D_out) {
    const cplx* phi = (const cplx*)phi_in;
    cplx* S = (cplx*)S_out;
    cplx* D = (cplx*)D_out;
#pragma omp parallel for schedule(dynamic, 32)
    for (int l = 0; l < o->n; ++l) {
        cplx as = 0, ad = 0, g, dg;
        const int tb = o->leaf_of[l];
        for (int j = o->nb_ptr[tb]; j < o->nb_ptr[tb + 1]; ++j) {
            const int b = o->nb_idx[j];
            for (uint32_t t = o->leaf_beg[b]; t < o->leaf_end[b]; ++t) {
                const int m = (int)o->perm[t];
                if (m == l) continue;
                int sing = 0;
                for (uint32_t p = o->tpb[l]; p < o->tpb[l + 1]; ++p) sing |= (o->pair_patch[p] == o->patch_of[m]);
                if (sing) continue;
                const cplx a = phi[m] * o->jw[m];
                kernels(o, l, m, &g, &dg);
                as += g * a;
                ad += dg * a;
            }
        }
        for (uint32_t p = o->tpb[l]; p < o->tpb[l + 1]; ++p)
            for (uint32_t f = o->far_begin[p]; f < o->far_end[p]; ++f) {
                const int m = (int)o->far_nodes[f];
                const cplx a = phi[m] * o->jw[m];
                kernels(o, l, m, &g, &dg);
                as -= g * a;
                ad -= dg * a;
            }
        S[l] += as;
        D[l] += ad;
    }
    return 0;
}

/* ------------------------------------------------------------ RP (rp.cpp:400-451) */
int oracle_rp_apply(int n, int npatch, const int32_t* nu, const int32_t* nv, const int64_t* patch_start,
                    const uint32_t* tpb, const int32_t* pair_patch, const uint64_t* beta_off,
                    const double* beta_s_in, const double* beta_d_in, const double* phi_in, double* S_out,
                    double* D_out) {
    const cplx* phi = (const cplx*)phi_in;
    const cplx* bs = (const cplx*)beta_s_in;
    const cplx* bd = (const cplx*)beta_d_in;
    cplx* S = (cplx*)S_out;
    cplx* D = (cplx*)D_out;
    cplx* coeff = calloc((size_t)patch_start[npatch] + 1, sizeof(cplx));
#pragma omp parallel for schedule(static)
    for (int q = 0; q < npatch; ++q) { /* coeffs_2d: along u per row, then along v per column */
        const int U = nu[q], V = nv[q];
        double xu[64], xv[64], t[64];
        cheb_nodes(U, xu);
        cheb_nodes(V, xv);
        cplx* tmp = calloc((size_t)U * V, sizeof(cplx));
        const cplx* s = phi + patch_start[q];
        for (int j = 0; j < V; ++j)
            for (int kk = 0; kk < U; ++kk) {
                t[0] = 1.0;
                if (U > 1) t[1] = xu[kk];
                for (int i = 2; i < U; ++i) t[i] = 2.0 * xu[kk] * t[i - 1] - t[i - 2];
                for (int i = 0; i < U; ++i) tmp[i + U * j] += s[kk + U * j] * t[i];
            }
        for (int j = 0; j < V; ++j)
            for (int i = 0; i < U; ++i) tmp[i + U * j] *= (i == 0 ? 1.0 : 2.0) / U;
        cplx* out = coeff + patch_start[q];
        for (int i = 0; i < U; ++i)
            for (int kk = 0; kk < V; ++kk) {
                t[0] = 1.0;
                if (V > 1) t[1] = xv[kk];
                for (int j = 2; j < V; ++j) t[j] = 2.0 * xv[kk] * t[j - 1] - t[j - 2];
                for (int j = 0; j < V; ++j) out[i + U * j] += tmp[i + U * kk] * t[j];
            }
        for (int i = 0; i < U; ++i)
            for (int j = 0; j < V; ++j) out[i + U * j] *= (j == 0 ? 1.0 : 2.0) / V;
        free(tmp);
    }
#pragma omp parallel for schedule(static)
    for (int l = 0; l < n; ++l)
        for (uint32_t p = tpb[l]; p < tpb[l + 1]; ++p) {
            const int q = pair_patch[p];
            const size_t nn = (size_t)nu[q] * nv[q];
            const cplx* a = coeff + patch_start[q];
            cplx as = 0, ad = 0;
            for (size_t i = 0; i < nn; ++i) {
                as += a[i] * bs[beta_off[p] + i];
                ad += a[i] * bd[beta_off[p] + i];
            }
            S[l] += as;
            D[l] += ad;
        }
    free(coeff);
    return 0;
}
