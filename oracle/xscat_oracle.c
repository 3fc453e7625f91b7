/*
 * xscat_oracle.c — TEST INFRASTRUCTURE ONLY (see xscat_oracle.h).
 *
 * Plain-C restatement of the reference projector path.  Each function cites
 * the reference file:line it restates (paths relative to
 * /root/reference/proj).  Expression order follows the reference so that,
 * compiled with -ffp-contract=off against the same libm, results are
 * bit-identical to the reference library (checked by tests/test_oracle.py
 * against oracle/_ref and tests/golden/).
 */
#define _GNU_SOURCE
#include "xscat_oracle.h"

#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* constants.hpp:9-22 */
#define XO_R0_CM 2.8179403e-13
#define XO_MEC2_KEV 511.0
#define XO_HC_KEV_A 12.398
#define XO_BARN_CM2 1.0e-24
#define XO_PI 3.14159265358979323846

/* ------------------------------------------------------------ error model */

typedef struct xo_err {
    jmp_buf jb;
    int code;
    char msg[512];
} xo_err;

static __thread xo_err* tl_err = NULL;
static __thread char tl_last[512];

static void xo_throw(int code, const char* fmt, ...)
{
    va_list ap;
    xo_err* e = tl_err;
    va_start(ap, fmt);
    if (e) {
        vsnprintf(e->msg, sizeof e->msg, fmt, ap);
        e->code = code;
        va_end(ap);
        longjmp(e->jb, 1);
    }
    vsnprintf(tl_last, sizeof tl_last, fmt, ap);
    va_end(ap);
    abort();
}

const char* xo_last_error(void) { return tl_last; }

#define XO_TRY                                                                                 \
    xo_err err__;                                                                              \
    xo_err* prev__ = tl_err;                                                                   \
    tl_err = &err__;                                                                           \
    if (setjmp(err__.jb)) {                                                                    \
        tl_err = prev__;                                                                       \
        snprintf(tl_last, sizeof tl_last, "%s", err__.msg);                                    \
        return err__.code;                                                                     \
    }
#define XO_END tl_err = prev__;

/* ------------------------------------------------------------------ RNG
 * rng.hpp:11-67: Philox4x32-10, key = seed, counter {block, photon, bin, angle}. */

typedef struct orng {
    uint32_t key[2];
    uint32_t base[4];
    uint32_t buf[4];
    uint32_t block;
    int pos;
} orng;

static void rng_init(orng* r, uint64_t seed, uint32_t angle, uint32_t bin, uint32_t photon)
{
    r->key[0] = (uint32_t)seed;
    r->key[1] = (uint32_t)(seed >> 32);
    r->base[0] = 0u;
    r->base[1] = photon;
    r->base[2] = bin;
    r->base[3] = angle;
    r->block = 0;
    r->pos = 4;
}

static void rng_refill(orng* r) /* rng.hpp:44-60 */
{
    uint32_t c0 = r->block, c1 = r->base[1], c2 = r->base[2], c3 = r->base[3];
    uint32_t k0 = r->key[0], k1 = r->key[1];
    int round;
    for (round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
        const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    r->buf[0] = c0;
    r->buf[1] = c1;
    r->buf[2] = c2;
    r->buf[3] = c3;
    r->pos = 0;
    ++r->block;
}

static uint32_t rng_u32(orng* r)
{
    if (r->pos == 4)
        rng_refill(r);
    return r->buf[r->pos++];
}

static double rng_uniform(orng* r) /* rng.hpp:29-35 */
{
    const uint64_t hi = rng_u32(r);
    const uint64_t lo = rng_u32(r);
    const uint64_t bits = ((hi << 32) | lo) >> 11;
    return ((double)bits + 0.5) * 0x1p-53;
}

void xo_rng_uniform(uint64_t seed, uint32_t angle, uint32_t bin, uint32_t photon, int64_t n,
                    double* out)
{
    orng r;
    int64_t i;
    rng_init(&r, seed, angle, bin, photon);
    for (i = 0; i < n; ++i)
        out[i] = rng_uniform(&r);
}

void xo_rng_u32(uint64_t seed, uint32_t angle, uint32_t bin, uint32_t photon, int64_t n,
                uint32_t* out)
{
    orng r;
    int64_t i;
    rng_init(&r, seed, angle, bin, photon);
    for (i = 0; i < n; ++i)
        out[i] = rng_u32(&r);
}

/* ---------------------------------------------------------------- tables
 * table.hpp:38-91 */

static void tab_locate(const xs_table* t, double x, int* idx, int* exact)
{
    int lo = 0, hi = t->n - 1;
    if (!(x >= t->x[0] && x <= t->x[t->n - 1]))
        xo_throw(XS_E_OUT_OF_RANGE, "table: query %f outside [%f, %f]", x, t->x[0],
                 t->x[t->n - 1]);
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (t->x[mid] <= x)
            lo = mid;
        else
            hi = mid;
    }
    if (x == t->x[lo]) {
        *idx = lo;
        *exact = 1;
        return;
    }
    if (x == t->x[hi]) {
        *idx = hi;
        *exact = 1;
        return;
    }
    *idx = lo;
    *exact = 0;
}

static double tab_linear(const xs_table* t, double x)
{
    int i, ex;
    double u;
    tab_locate(t, x, &i, &ex);
    if (ex)
        return t->y[i];
    u = (x - t->x[i]) / (t->x[i + 1] - t->x[i]);
    return t->y[i] + u * (t->y[i + 1] - t->y[i]);
}

static double tab_linear_clamped(const xs_table* t, double x)
{
    if (x <= t->x[0])
        return t->y[0];
    if (x >= t->x[t->n - 1])
        return t->y[t->n - 1];
    return tab_linear(t, x);
}

static double tab_loglog(const xs_table* t, double x)
{
    int i, ex;
    double u;
    tab_locate(t, x, &i, &ex);
    if (ex)
        return t->y[i];
    if (t->y[i] <= 0.0 || t->y[i + 1] <= 0.0) {
        u = (x - t->x[i]) / (t->x[i + 1] - t->x[i]);
        return t->y[i] + u * (t->y[i + 1] - t->y[i]);
    }
    u = (log(x) - log(t->x[i])) / (log(t->x[i + 1]) - log(t->x[i]));
    return exp(log(t->y[i]) + u * (log(t->y[i + 1]) - log(t->y[i])));
}

int xo_table_eval(const xs_table* t, int32_t mode, double x, double* y)
{
    XO_TRY
    *y = mode == 0 ? tab_linear(t, x) : mode == 1 ? tab_linear_clamped(t, x) : tab_loglog(t, x);
    XO_END
    return XS_OK;
}

/* -------------------------------------------------------------- materials */

typedef struct omat {
    const xs_material* m;
    double* cdf; /* f2_q2_cdf, material.cpp:107-125 */
    int has_tables;
} omat;

static void build_cdf(const xs_material* m, double* cdf) /* material.cpp:107-125 */
{
    const double* q = m->f_factor.x;
    const double* fv = m->f_factor.y;
    int i;
    cdf[0] = 0.0;
    for (i = 1; i < m->f_factor.n; ++i) {
        const double q0 = q[i - 1], q1 = q[i];
        const double a = fv[i - 1];
        const double b = (fv[i] - fv[i - 1]) / (q1 - q0);
        const double h = q1 - q0;
        const double c0 = a * a, c1 = 2.0 * a * b, c2 = b * b;
        const double integral = 2.0 * (c0 * q0 * h + (c0 + c1 * q0) * h * h / 2.0 +
                                       (c1 + c2 * q0) * h * h * h / 3.0 +
                                       c2 * h * h * h * h / 4.0);
        cdf[i] = cdf[i - 1] + integral;
    }
}

int xo_f2_q2_cdf(const xs_material* m, double* out)
{
    build_cdf(m, out);
    return XS_OK;
}

static void omat_init(omat* o, const xs_material* m)
{
    o->m = m;
    o->has_tables = m->mu.n > 0;
    o->cdf = NULL;
    if (o->has_tables && m->f_factor.n > 0) {
        o->cdf = (double*)malloc(sizeof(double) * (size_t)m->f_factor.n);
        build_cdf(m, o->cdf);
    }
}

static void omat_free(omat* o) { free(o->cdf); }

/* material.cpp:253-271 */
static double form_factor_S(const omat* o, double q)
{
    const xs_material* m = o->m;
    if (!(q >= 0.0))
        xo_throw(XS_E_DOMAIN, "form_factor_S: negative q");
    if (q >= m->s_factor.x[m->s_factor.n - 1])
        return m->z_eff;
    return tab_linear(&m->s_factor, q);
}

static double form_factor_F(const omat* o, double q)
{
    if (!(q >= 0.0))
        xo_throw(XS_E_DOMAIN, "form_factor_F: negative q");
    return tab_linear_clamped(&o->m->f_factor, q);
}

/* ---------------------------------------------------------- cross sections
 * cross_sections.cpp:11-96 */

static void check_theta(double theta)
{
    if (!(theta >= 0.0 && theta <= XO_PI))
        xo_throw(XS_E_DOMAIN, "scatter angle outside [0, pi]");
}

static double momentum_transfer(double e, double theta)
{
    return sin(0.5 * theta) * e / XO_HC_KEV_A;
}

static double compton_energy_ratio(double e, double theta)
{
    const double alpha = e / XO_MEC2_KEV;
    return 1.0 / (1.0 + alpha * (1.0 - cos(theta)));
}

static double kn_core(double e, double theta)
{
    const double ratio = compton_energy_ratio(e, theta);
    const double s = sin(theta);
    return ratio * ratio * (ratio + 1.0 / ratio - s * s);
}

static double p_lambda_compton(const omat* o, double e, double theta)
{
    double sigma, r0;
    check_theta(theta);
    sigma = tab_loglog(&o->m->sigma_incoh, e) * XO_BARN_CM2;
    if (!(sigma > 0.0))
        xo_throw(XS_E_RUNTIME, "p_lambda_compton: vanishing incoherent cross section at %f keV",
                 e);
    r0 = XO_R0_CM;
    return XO_PI * r0 * r0 / sigma * kn_core(e, theta) *
           form_factor_S(o, momentum_transfer(e, theta));
}

static double p_lambda_rayleigh(const omat* o, double e, double theta)
{
    double sigma, r0, c, f;
    check_theta(theta);
    sigma = tab_loglog(&o->m->sigma_coh, e) * XO_BARN_CM2;
    if (!(sigma > 0.0))
        xo_throw(XS_E_RUNTIME, "p_lambda_rayleigh: vanishing coherent cross section at %f keV",
                 e);
    r0 = XO_R0_CM;
    c = cos(theta);
    f = form_factor_F(o, momentum_transfer(e, theta));
    return XO_PI * r0 * r0 / sigma * (1.0 + c * c) * f * f;
}

static double d_sigma_compton(const omat* o, double e, double theta)
{
    const double r0 = XO_R0_CM;
    check_theta(theta);
    return 0.5 * r0 * r0 * kn_core(e, theta) * form_factor_S(o, momentum_transfer(e, theta));
}

static double d_sigma_rayleigh(const omat* o, double e, double theta)
{
    const double r0 = XO_R0_CM;
    double c, f;
    check_theta(theta);
    c = cos(theta);
    f = form_factor_F(o, momentum_transfer(e, theta));
    return 0.5 * r0 * r0 * (1.0 + c * c) * f * f;
}

enum { K_PE = 0, K_COMPTON = 1, K_RAYLEIGH = 2 };

static int select_interaction(const omat* o, double e, orng* rng) /* :81-96 */
{
    const double pe = tab_loglog(&o->m->sigma_pe, e);
    const double incoh = tab_loglog(&o->m->sigma_incoh, e);
    const double coh = tab_loglog(&o->m->sigma_coh, e);
    const double total = pe + incoh + coh;
    double u;
    if (!(total > 0.0))
        xo_throw(XS_E_RUNTIME, "select_interaction: all cross sections vanish at %f keV in %s",
                 e, o->m->name ? o->m->name : "?");
    u = rng_uniform(rng) * total;
    if (u < pe)
        return K_PE;
    if (u < pe + incoh)
        return K_COMPTON;
    return K_RAYLEIGH;
}

/* ---------------------------------------------------------------- samplers
 * samplers.cpp:12-134 */

static double kahn_cos_theta(double alpha, orng* rng)
{
    const double t = 1.0 + 2.0 * alpha;
    for (;;) {
        const double r1 = rng_uniform(rng);
        const double r2 = rng_uniform(rng);
        const double r3 = rng_uniform(rng);
        if (r1 <= t / (t + 8.0)) {
            const double x = 1.0 + 2.0 * alpha * r2;
            if (r3 <= 4.0 * (1.0 / x - 1.0 / (x * x)))
                return 1.0 - (x - 1.0) / alpha;
        } else {
            const double x = t / (1.0 + 2.0 * alpha * r2);
            const double cos_th = 1.0 - (x - 1.0) / alpha;
            if (r3 <= 0.5 * (cos_th * cos_th + 1.0 / x))
                return cos_th;
        }
    }
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

static void sample_compton(const omat* o, double e, orng* rng, double* theta_out,
                           double* alpha_prime, double* phi)
{
    const double alpha = e / XO_MEC2_KEV;
    const double q_max = momentum_transfer(e, XO_PI);
    const double s_max = form_factor_S(o, q_max);
    if (!(s_max > 0.0))
        xo_throw(XS_E_RUNTIME, "sample_compton: S vanishes over the kinematic range at %f keV",
                 e);
    for (;;) {
        const double cos_th = kahn_cos_theta(alpha, rng);
        const double theta = acos(clampd(cos_th, -1.0, 1.0));
        const double s = form_factor_S(o, momentum_transfer(e, theta));
        if (rng_uniform(rng) * s_max <= s) {
            *theta_out = theta;
            *alpha_prime = alpha / (1.0 + alpha * (1.0 - cos(theta)));
            *phi = 2.0 * XO_PI * rng_uniform(rng);
            return;
        }
    }
}

static double segment_mass(double q0, double a, double b, double u) /* :56-62 */
{
    const double c0 = a * a, c1 = 2.0 * a * b, c2 = b * b;
    return 2.0 * (c0 * q0 * u + (c0 + c1 * q0) * u * u / 2.0 +
                  (c1 + c2 * q0) * u * u * u / 3.0 + c2 * u * u * u * u / 4.0);
}

static double cumulative_mass(const omat* o, double q) /* :64-88 */
{
    const double* knots = o->m->f_factor.x;
    const double* fv = o->m->f_factor.y;
    const int n = o->m->f_factor.n;
    int lo = 0, hi = n - 1;
    double a, b;
    if (q >= knots[n - 1]) {
        const double f_last = fv[n - 1];
        return o->cdf[n - 1] + f_last * f_last * (q * q - knots[n - 1] * knots[n - 1]);
    }
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (knots[mid] <= q)
            lo = mid;
        else
            hi = mid;
    }
    a = fv[lo];
    b = (fv[lo + 1] - fv[lo]) / (knots[lo + 1] - knots[lo]);
    return o->cdf[lo] + segment_mass(knots[lo], a, b, q - knots[lo]);
}

static double invert_mass(const omat* o, double target, double q_hi) /* :92-102 */
{
    double lo = 0.0, hi = q_hi;
    int it;
    for (it = 0; it < 64; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (cumulative_mass(o, mid) < target)
            lo = mid;
        else
            hi = mid;
    }
    return 0.5 * (lo + hi);
}

static void sample_rayleigh(const omat* o, double e, orng* rng, double* theta_out, double* phi)
{
    const double q_max = momentum_transfer(e, XO_PI);
    const double total = cumulative_mass(o, q_max);
    double scale;
    if (!(total > 0.0))
        xo_throw(XS_E_RUNTIME, "sample_rayleigh: F vanishes over the kinematic range at %f keV",
                 e);
    scale = XO_HC_KEV_A / e;
    for (;;) {
        const double q = invert_mass(o, rng_uniform(rng) * total, q_max);
        const double sh = q * scale < 1.0 ? q * scale : 1.0;
        const double cos_th = 1.0 - 2.0 * sh * sh;
        if (rng_uniform(rng) * 2.0 <= 1.0 + cos_th * cos_th) {
            *theta_out = acos(clampd(cos_th, -1.0, 1.0));
            *phi = 2.0 * XO_PI * rng_uniform(rng);
            return;
        }
    }
}

typedef struct v3 {
    double x, y, z;
} v3;

static v3 v3m(double x, double y, double z)
{
    v3 r;
    r.x = x;
    r.y = y;
    r.z = z;
    return r;
}
static v3 vadd(v3 a, v3 b) { return v3m(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return v3m(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, double s) { return v3m(a.x * s, a.y * s, a.z * s); }
static v3 vdiv(v3 a, double s) { return v3m(a.x / s, a.y / s, a.z / s); }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b)
{
    return v3m(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static v3 vnormalized(v3 v) { return vdiv(v, sqrt(vdot(v, v))); }

static v3 rotate_direction(v3 dir, double theta, double phi) /* samplers.cpp:127-134 */
{
    const v3 pick = fabs(dir.x) < 0.5 ? v3m(1.0, 0.0, 0.0) : v3m(0.0, 1.0, 0.0);
    const v3 e1 = vnormalized(vcross(dir, pick));
    const v3 e2 = vcross(dir, e1);
    const double st = sin(theta), ct = cos(theta);
    return vnormalized(vadd(vmul(dir, ct), vmul(vadd(vmul(e1, cos(phi)), vmul(e2, sin(phi))), st)));
}

void xo_rotate_direction(const double dir[3], double theta, double phi, double out[3])
{
    const v3 r = rotate_direction(v3m(dir[0], dir[1], dir[2]), theta, phi);
    out[0] = r.x;
    out[1] = r.y;
    out[2] = r.z;
}

/* ----------------------------------------------------------------- scene */

typedef struct oscene {
    const xs_phantom* ph;
    omat* mats;
    int n_mats;
} oscene;

static void scene_init(oscene* s, const xs_phantom* ph)
{
    int i;
    s->ph = ph;
    s->n_mats = ph->n_materials;
    s->mats = (omat*)calloc((size_t)ph->n_materials, sizeof(omat));
    for (i = 0; i < ph->n_materials; ++i) {
        if (i == 0) {
            s->mats[i].m = &ph->materials[0];
            s->mats[i].has_tables = 0;
            continue;
        }
        omat_init(&s->mats[i], &ph->materials[i]);
    }
}

static void scene_free(oscene* s)
{
    int i;
    for (i = 0; i < s->n_mats; ++i)
        omat_free(&s->mats[i]);
    free(s->mats);
}

/* MuField (trace.cpp:10-16): mass attenuation per material id at E. */
static void mu_field(const oscene* s, double e, double* mass_atten)
{
    int i;
    mass_atten[0] = 0.0;
    for (i = 1; i < s->n_mats; ++i)
        mass_atten[i] = s->mats[i].has_tables ? tab_loglog(&s->mats[i].m->mu, e) : 0.0;
}

static size_t cell_index(const xs_phantom* ph, int ix, int iy, int iz)
{
    return (size_t)ix + (size_t)ph->dims[0] * ((size_t)iy + (size_t)ph->dims[1] * (size_t)iz);
}

static double mu_at_cell(const xs_phantom* ph, const double* mass_atten, size_t cell)
{
    return mass_atten[ph->material_id[cell]] * (double)ph->density[cell];
}

/* ----------------------------------------------------------------- tracing
 * trace.cpp:22-230 */

static int finite3(v3 v) { return isfinite(v.x) && isfinite(v.y) && isfinite(v.z); }

static int clip_to_grid(const xs_phantom* ph, v3 ro, v3 rd, double* t_enter, double* t_exit)
{
    const double o[3] = {ro.x, ro.y, ro.z};
    const double d[3] = {rd.x, rd.y, rd.z};
    double l[3], h[3];
    double t0 = 0.0, t1 = INFINITY;
    int a;
    if (!finite3(ro) || !finite3(rd))
        xo_throw(XS_E_INVALID_ARGUMENT, "trace: non-finite ray");
    for (a = 0; a < 3; ++a) {
        l[a] = ph->origin[a];
        h[a] = ph->origin[a] + ph->dims[a] * ph->voxel_size[a];
    }
    for (a = 0; a < 3; ++a) {
        double ta, tb;
        if (d[a] == 0.0) {
            if (o[a] < l[a] || o[a] >= h[a])
                return 0;
            continue;
        }
        ta = (l[a] - o[a]) / d[a];
        tb = (h[a] - o[a]) / d[a];
        if (ta > tb) {
            const double tmp = ta;
            ta = tb;
            tb = tmp;
        }
        t0 = t0 > ta ? t0 : ta;
        t1 = tb < t1 ? tb : t1;
    }
    if (!(t0 < t1))
        return 0;
    *t_enter = t0;
    *t_exit = t1;
    return 1;
}

typedef struct owalk {
    int idx[3];
    int step[3];
    double t_next[3];
    double dt[3];
} owalk;

static int voxel_of(double p, double org, double inv_h, int n)
{
    int i = (int)floor((p - org) * inv_h);
    return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

static void start_walk(const xs_phantom* ph, v3 ro, v3 rd, double t0, owalk* w)
{
    const v3 p = vadd(ro, vmul(rd, t0));
    const double o[3] = {ro.x, ro.y, ro.z};
    const double d[3] = {rd.x, rd.y, rd.z};
    const double pp[3] = {p.x, p.y, p.z};
    int a;
    for (a = 0; a < 3; ++a) {
        const double org = ph->origin[a], hs = ph->voxel_size[a];
        w->idx[a] = voxel_of(pp[a], org, 1.0 / hs, ph->dims[a]);
        if (d[a] > 0.0) {
            w->step[a] = 1;
            w->dt[a] = hs / d[a];
            w->t_next[a] = (org + (w->idx[a] + 1) * hs - o[a]) / d[a];
        } else if (d[a] < 0.0) {
            w->step[a] = -1;
            w->dt[a] = -hs / d[a];
            w->t_next[a] = (org + w->idx[a] * hs - o[a]) / d[a];
        } else {
            w->step[a] = 0;
            w->dt[a] = INFINITY;
            w->t_next[a] = INFINITY;
        }
        while (w->t_next[a] <= t0 && w->step[a] != 0) {
            w->idx[a] += w->step[a];
            w->t_next[a] += w->dt[a];
        }
    }
}

static double min4(double a, double b, double c, double d)
{
    double m = a;
    if (b < m)
        m = b;
    if (c < m)
        m = c;
    if (d < m)
        m = d;
    return m;
}

/* trace_attenuation (trace.cpp:107-155); *steps counts voxel visits. */
static double trace_attenuation(const xs_phantom* ph, v3 ro, v3 rd, const double* mass_atten,
                                int step_voxels, uint64_t* steps)
{
    double te, tx, depth, t;
    owalk w;
    if (step_voxels < 1)
        xo_throw(XS_E_INVALID_ARGUMENT, "trace_attenuation: step_voxels must be >= 1");
    if (!clip_to_grid(ph, ro, rd, &te, &tx))
        return 0.0;
    if (step_voxels > 1) {
        double vmin = ph->voxel_size[0];
        double h, len, ihx, ihy, ihz;
        int n, j;
        if (ph->voxel_size[1] < vmin)
            vmin = ph->voxel_size[1];
        if (ph->voxel_size[2] < vmin)
            vmin = ph->voxel_size[2];
        h = step_voxels * vmin;
        len = tx - te;
        n = (int)ceil(len / h);
        if (n < 1)
            n = 1;
        ihx = 1.0 / ph->voxel_size[0];
        ihy = 1.0 / ph->voxel_size[1];
        ihz = 1.0 / ph->voxel_size[2];
        depth = 0.0;
        for (j = 0; j < n; ++j) {
            const double ta = te + j * h;
            const double tb = ta + h < tx ? ta + h : tx;
            const v3 p = vadd(ro, vmul(rd, 0.5 * (ta + tb)));
            const int ix = voxel_of(p.x, ph->origin[0], ihx, ph->dims[0]);
            const int iy = voxel_of(p.y, ph->origin[1], ihy, ph->dims[1]);
            const int iz = voxel_of(p.z, ph->origin[2], ihz, ph->dims[2]);
            depth += mu_at_cell(ph, mass_atten, cell_index(ph, ix, iy, iz)) * (tb - ta);
        }
        if (steps)
            *steps += (uint64_t)n;
        return depth;
    }
    start_walk(ph, ro, rd, te, &w);
    depth = 0.0;
    t = te;
    while (t < tx) {
        const double tn = min4(w.t_next[0], w.t_next[1], w.t_next[2], tx);
        int a;
        if (steps)
            ++*steps;
        depth += mu_at_cell(ph, mass_atten, cell_index(ph, w.idx[0], w.idx[1], w.idx[2])) *
                 (tn - t);
        t = tn;
        if (t >= tx)
            break;
        for (a = 0; a < 3; ++a) {
            if (w.t_next[a] == tn) {
                w.idx[a] += w.step[a];
                if (w.idx[a] < 0 || w.idx[a] >= ph->dims[a])
                    return depth;
                w.t_next[a] += w.dt[a];
            }
        }
    }
    return depth;
}

/* trace_rho_lengths (trace.cpp:163-187) */
static void trace_rho_lengths(const xs_phantom* ph, v3 ro, v3 rd, double* out)
{
    double te, tx, t;
    owalk w;
    int m;
    for (m = 0; m < ph->n_materials; ++m)
        out[m] = 0.0;
    if (!clip_to_grid(ph, ro, rd, &te, &tx))
        return;
    start_walk(ph, ro, rd, te, &w);
    t = te;
    while (t < tx) {
        const double tn = min4(w.t_next[0], w.t_next[1], w.t_next[2], tx);
        const size_t cell = cell_index(ph, w.idx[0], w.idx[1], w.idx[2]);
        int a;
        out[ph->material_id[cell]] += (double)ph->density[cell] * (tn - t);
        t = tn;
        if (t >= tx)
            break;
        for (a = 0; a < 3; ++a) {
            if (w.t_next[a] == tn) {
                w.idx[a] += w.step[a];
                if (w.idx[a] < 0 || w.idx[a] >= ph->dims[a])
                    return;
                w.t_next[a] += w.dt[a];
            }
        }
    }
}

typedef struct ofp {
    int escaped;
    v3 point;
    int ix, iy, iz;
} ofp;

/* sample_free_path (trace.cpp:189-230) */
static ofp sample_free_path(const xs_phantom* ph, v3 ro, v3 rd, const double* mass_atten,
                            double u, uint64_t* steps)
{
    ofp r;
    double target, te, tx, depth, t;
    owalk w;
    r.escaped = 1;
    r.point = v3m(0, 0, 0);
    r.ix = r.iy = r.iz = 0;
    if (!(u > 0.0 && u < 1.0))
        xo_throw(XS_E_INVALID_ARGUMENT, "sample_free_path: u must lie in (0,1)");
    target = -log(u);
    if (!clip_to_grid(ph, ro, rd, &te, &tx))
        return r;
    start_walk(ph, ro, rd, te, &w);
    depth = 0.0;
    t = te;
    while (t < tx) {
        const double tn = min4(w.t_next[0], w.t_next[1], w.t_next[2], tx);
        const double mu_cell =
            mu_at_cell(ph, mass_atten, cell_index(ph, w.idx[0], w.idx[1], w.idx[2]));
        const double seg = mu_cell * (tn - t);
        int a;
        if (steps)
            ++*steps;
        if (depth + seg >= target) {
            const double t_hit = (mu_cell > 0.0) ? t + (target - depth) / mu_cell : tn;
            r.escaped = 0;
            r.point = vadd(ro, vmul(rd, t_hit));
            r.ix = w.idx[0];
            r.iy = w.idx[1];
            r.iz = w.idx[2];
            return r;
        }
        depth += seg;
        t = tn;
        if (t >= tx)
            break;
        for (a = 0; a < 3; ++a) {
            if (w.t_next[a] == tn) {
                w.idx[a] += w.step[a];
                if (w.idx[a] < 0 || w.idx[a] >= ph->dims[a])
                    return r;
                w.t_next[a] += w.dt[a];
            }
        }
    }
    return r;
}

/* ------------------------------------------------ public tracing wrappers */

int xo_trace_attenuation(const xs_phantom* ph, const double origin[3], const double dir[3],
                         double energy_kev, int32_t step_voxels, double* tau)
{
    oscene s;
    double ma[256];
    XO_TRY
    scene_init(&s, ph);
    mu_field(&s, energy_kev, ma);
    *tau = trace_attenuation(ph, v3m(origin[0], origin[1], origin[2]),
                             v3m(dir[0], dir[1], dir[2]), ma, step_voxels, NULL);
    scene_free(&s);
    XO_END
    return XS_OK;
}

int xo_trace_rho_lengths(const xs_phantom* ph, const double origin[3], const double dir[3],
                         double* rho_len)
{
    XO_TRY
    trace_rho_lengths(ph, v3m(origin[0], origin[1], origin[2]), v3m(dir[0], dir[1], dir[2]),
                      rho_len);
    XO_END
    return XS_OK;
}

int xo_sample_free_path(const xs_phantom* ph, const double origin[3], const double dir[3],
                        double energy_kev, double u, int32_t* escaped, double point[3],
                        int32_t voxel[3])
{
    oscene s;
    double ma[256];
    ofp r;
    XO_TRY
    scene_init(&s, ph);
    mu_field(&s, energy_kev, ma);
    r = sample_free_path(ph, v3m(origin[0], origin[1], origin[2]), v3m(dir[0], dir[1], dir[2]),
                         ma, u, NULL);
    scene_free(&s);
    XO_END
    *escaped = r.escaped;
    point[0] = r.point.x;
    point[1] = r.point.y;
    point[2] = r.point.z;
    voxel[0] = r.ix;
    voxel[1] = r.iy;
    voxel[2] = r.iz;
    return XS_OK;
}

/* ------------------------------------------------ public sampler wrappers */

int xo_p_lambda(const xs_material* m, int32_t compton, double e, double theta, double* p)
{
    omat o;
    XO_TRY
    omat_init(&o, m);
    *p = compton ? p_lambda_compton(&o, e, theta) : p_lambda_rayleigh(&o, e, theta);
    omat_free(&o);
    XO_END
    return XS_OK;
}

int xo_d_sigma(const xs_material* m, int32_t compton, double e, double theta, double* d)
{
    omat o;
    XO_TRY
    omat_init(&o, m);
    *d = compton ? d_sigma_compton(&o, e, theta) : d_sigma_rayleigh(&o, e, theta);
    omat_free(&o);
    XO_END
    return XS_OK;
}

int xo_sample_compton(const xs_material* m, double e, uint64_t seed, int64_t n, double* theta,
                      double* phi, double* alpha_prime)
{
    omat o;
    orng r;
    int64_t i;
    XO_TRY
    omat_init(&o, m);
    rng_init(&r, seed, 0, 0, 0);
    for (i = 0; i < n; ++i) {
        double th, ap, ph;
        sample_compton(&o, e, &r, &th, &ap, &ph);
        theta[i] = th;
        if (phi)
            phi[i] = ph;
        if (alpha_prime)
            alpha_prime[i] = ap;
    }
    omat_free(&o);
    XO_END
    return XS_OK;
}

int xo_sample_rayleigh(const xs_material* m, double e, uint64_t seed, int64_t n, double* theta,
                       double* phi)
{
    omat o;
    orng r;
    int64_t i;
    XO_TRY
    omat_init(&o, m);
    rng_init(&r, seed, 0, 0, 0);
    for (i = 0; i < n; ++i) {
        double th, ph;
        sample_rayleigh(&o, e, &r, &th, &ph);
        theta[i] = th;
        if (phi)
            phi[i] = ph;
    }
    omat_free(&o);
    XO_END
    return XS_OK;
}

int xo_kahn_cos_theta(double alpha, uint64_t seed, int64_t n, double* out)
{
    orng r;
    int64_t i;
    rng_init(&r, seed, 0, 0, 0);
    for (i = 0; i < n; ++i)
        out[i] = kahn_cos_theta(alpha, &r);
    return XS_OK;
}

int xo_select_interaction(const xs_material* m, double e, uint64_t seed, int64_t n,
                          int32_t* kinds)
{
    omat o;
    orng r;
    int64_t i;
    XO_TRY
    omat_init(&o, m);
    rng_init(&r, seed, 0, 0, 0);
    for (i = 0; i < n; ++i)
        kinds[i] = select_interaction(&o, e, &r);
    omat_free(&o);
    XO_END
    return XS_OK;
}

/* --------------------------------------------------------------- geometry
 * scan_geometry.cpp:44-77 */

typedef struct oframe {
    v3 src, center, uaxis, normal;
} oframe;

static oframe frame_of(const xs_geometry* g, int angle_idx)
{
    oframe f;
    const double a = g->angles[angle_idx];
    const double r = g->sdd - g->sod;
    f.src = v3m(g->sod * cos(a), g->sod * sin(a), 0.0);
    f.center = v3m(-r * cos(a), -r * sin(a), 0.0);
    f.uaxis = v3m(-sin(a), cos(a), 0.0);
    f.normal = v3m(cos(a), sin(a), 0.0);
    return f;
}

static v3 pixel_position(const xs_geometry* g, const oframe* f, double u, double v)
{
    const v3 va = v3m(0.0, 0.0, 1.0);
    const double du = (u + 0.5 - 0.5 * g->nu) * g->pixel_pitch;
    const double dv = (v + 0.5 - 0.5 * g->nv) * g->pixel_pitch;
    return vadd(vadd(f->center, vmul(f->uaxis, du)), vmul(va, dv));
}

static void validate_geometry(const xs_geometry* g) /* scan_geometry.cpp:9-26 */
{
    int i;
    if (!(g->sod > 0.0 && g->sdd > g->sod))
        xo_throw(XS_E_RUNTIME, "geometry: require 0 < sod < sdd");
    if (g->nu <= 0 || g->nv <= 0)
        xo_throw(XS_E_RUNTIME, "geometry: detector pixel counts must be positive");
    if (!(g->pixel_pitch > 0.0))
        xo_throw(XS_E_RUNTIME, "geometry: pixel pitch must be positive");
    if (g->n_angles <= 0)
        xo_throw(XS_E_RUNTIME, "geometry: no angles");
    for (i = 0; i < g->n_angles; ++i) {
        if (g->angles[i] < 0.0 || g->angles[i] >= 2.0 * XO_PI)
            xo_throw(XS_E_RUNTIME, "geometry: angles must lie in [0, 2pi)");
        if (i > 0 && !(g->angles[i] > g->angles[i - 1]))
            xo_throw(XS_E_RUNTIME, "geometry: angles must be strictly increasing");
    }
}

static void validate_spectrum(const xs_spectrum* s) /* spectrum.cpp:11-30 */
{
    double positive = 0.0;
    int i;
    if (s->n_bins <= 0)
        xo_throw(XS_E_RUNTIME, "spectrum: no bins");
    for (i = 0; i < s->n_bins; ++i) {
        if (!isfinite(s->energy_kev[i]) || !isfinite(s->weight[i]))
            xo_throw(XS_E_RUNTIME, "spectrum: non-finite entry");
        if (!(s->weight[i] >= 0.0))
            xo_throw(XS_E_RUNTIME, "spectrum: negative weight");
        if (i > 0 && !(s->energy_kev[i] > s->energy_kev[i - 1]))
            xo_throw(XS_E_RUNTIME, "spectrum: non-monotone abscissa");
        positive += s->weight[i];
    }
    if (!(positive > 0.0))
        xo_throw(XS_E_RUNTIME, "spectrum: all weights zero");
    if (s->energy_kev[0] < 1.0 || s->energy_kev[s->n_bins - 1] > 1000.0)
        xo_throw(XS_E_RUNTIME, "spectrum: energies must lie within [1 keV, 1 MeV]");
}

static void validate_sim_config(const xs_sim_config* c) /* transport.cpp:26-40 */
{
    if (c->photons_total < 1)
        xo_throw(XS_E_RUNTIME, "sim config: photons_total must be >= 1");
    if (c->splitting < 1)
        xo_throw(XS_E_RUNTIME, "sim config: splitting must be >= 1");
    if (!(c->roulette_survival > 0.0 && c->roulette_survival <= 1.0))
        xo_throw(XS_E_RUNTIME, "sim config: roulette_survival must lie in (0,1]");
    if (c->roulette_wmin_rel < 0.0)
        xo_throw(XS_E_RUNTIME, "sim config: roulette_wmin_rel must be >= 0");
    if (c->step_voxels < 1)
        xo_throw(XS_E_RUNTIME, "sim config: step_voxels must be >= 1");
    if (c->max_interactions < 1)
        xo_throw(XS_E_RUNTIME, "sim config: max_interactions must be >= 1");
}

/* ----------------------------------------------------- photon apportioning
 * transport.cpp:42-64 (stable sort on fractional parts, descending). */

typedef struct frac_ent {
    double f;
    int i;
} frac_ent;

int xo_apportion_photons(const xs_spectrum* spec, uint64_t photons_total, uint64_t* counts)
{
    double w_total = 0.0;
    const int n = spec->n_bins;
    frac_ent* fr = (frac_ent*)malloc(sizeof(frac_ent) * (size_t)(n > 0 ? n : 1));
    uint64_t assigned = 0;
    int i, k;
    for (i = 0; i < n; ++i)
        w_total += spec->weight[i];
    for (i = 0; i < n; ++i) {
        const double quota = photons_total * spec->weight[i] / w_total;
        counts[i] = (uint64_t)quota;
        assigned += counts[i];
        fr[i].f = quota - counts[i];
        fr[i].i = i;
    }
    /* stable insertion sort, descending by f */
    for (i = 1; i < n; ++i) {
        frac_ent cur = fr[i];
        int j = i - 1;
        while (j >= 0 && cur.f > fr[j].f) {
            fr[j + 1] = fr[j];
            --j;
        }
        fr[j + 1] = cur;
    }
    for (k = 0; assigned < photons_total && k < n; ++k, ++assigned)
        ++counts[fr[k].i];
    for (i = 0; i < n; ++i)
        if (spec->weight[i] > 0.0 && counts[i] == 0)
            counts[i] = 1;
    free(fr);
    return XS_OK;
}

/* --------------------------------------------------------------- transport */

typedef struct oledger {
    double initial, escaped, absorbed, culled, killed, boost;
} oledger;

typedef struct octx {
    oscene scene;
    const xs_phantom* ph;
    const xs_geometry* g;
    int angle_idx;
    oframe fr;
    const xs_spectrum* spec;
    const xs_response* resp;
    const xs_sim_config* cfg;
    uint64_t* photons_per_bin;
    xs_accum_units units;
} octx;

/* What a history produces; filled by run_history, consumed by a sink. */
typedef struct ohist_out {
    double total;
    int n_scores;
    int cap;
    size_t* pix;
    double* val;
    int n_led;               /* this history's ledger events, in order */
    int led_kind[128];       /* 0 initial 1 escaped 2 absorbed 3 culled 4 killed 5 boost */
    double led_val[128];
    uint64_t fp_steps, sc_steps, rays, interactions;
} ohist_out;

static void led_push(ohist_out* h, int kind, double v)
{
    if (h->n_led < 128) {
        h->led_kind[h->n_led] = kind;
        h->led_val[h->n_led] = v;
        ++h->n_led;
    }
}

static void hist_push(ohist_out* h, size_t pixel, double x)
{
    if (h->n_scores == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->pix = (size_t*)realloc(h->pix, sizeof(size_t) * (size_t)h->cap);
        h->val = (double*)realloc(h->val, sizeof(double) * (size_t)h->cap);
    }
    h->pix[h->n_scores] = pixel;
    h->val[h->n_scores] = x;
    ++h->n_scores;
}

static double response_factor(const xs_response* r, double e) /* detector_response.hpp:21-24 */
{
    return tab_linear(&r->deposit, e) / e;
}

/* point_detector_score (transport.cpp:66-71) */
static double pd_score(double rf, double p_dir, double w, double n_pixels, double d2, double tau)
{
    return rf * p_dir * w * n_pixels / (2.0 * XO_PI * d2) * exp(-tau);
}

/* run_history (transport.cpp:114-242). */
static void run_history(const octx* c, int bin, uint64_t photon, ohist_out* h)
{
    const xs_sim_config* cfg = c->cfg;
    const xs_geometry* g = c->g;
    const xs_phantom* ph = c->ph;
    const double bin_weight = c->spec->weight[bin];
    const double n_pixels = (double)g->nu * g->nv;
    orng rng;
    v3 pos, dir, delta, target;
    double energy, weight, w0, w_min, d2, xu, xv, cos_psi, em_weight;
    int generation = 0;
    double ma[256];

    h->n_scores = 0;
    h->total = 0.0;
    h->n_led = 0;

    rng_init(&rng, cfg->seed, (uint32_t)c->angle_idx, (uint32_t)bin, (uint32_t)photon);

    /* sample_emission (transport.cpp:73-87) */
    xu = (rng_uniform(&rng) - 0.5) * g->nu * g->pixel_pitch;
    xv = (rng_uniform(&rng) - 0.5) * g->nv * g->pixel_pitch;
    target = vadd(vadd(c->fr.center, vmul(c->fr.uaxis, xu)), vmul(v3m(0.0, 0.0, 1.0), xv));
    delta = vsub(target, c->fr.src);
    d2 = vdot(delta, delta);
    dir = vdiv(delta, sqrt(d2));
    cos_psi = -vdot(dir, c->fr.normal);
    em_weight = (double)(g->nu * g->nv) * g->pixel_pitch * g->pixel_pitch * cos_psi / d2;

    w0 = bin_weight * em_weight / (double)c->photons_per_bin[bin];
    w_min = cfg->roulette_wmin_rel * w0;
    pos = c->fr.src;
    energy = c->spec->energy_kev[bin];
    weight = w0;
    led_push(h, 0, w0);

    mu_field(&c->scene, energy, ma);
    for (;;) {
        const ofp fp = sample_free_path(ph, pos, dir, ma, rng_uniform(&rng), &h->fp_steps);
        const omat* mat;
        int kind, s;
        double w_split;
        if (fp.escaped) {
            led_push(h, 1, weight);
            break;
        }
        pos = fp.point;
        mat = &c->scene.mats[ph->material_id[cell_index(ph, fp.ix, fp.iy, fp.iz)]];
        ++h->interactions;
        kind = select_interaction(mat, energy, &rng);
        if (kind == K_PE) {
            led_push(h, 2, weight);
            break;
        }
        w_split = weight / cfg->splitting;
        for (s = 0; s < cfg->splitting; ++s) {
            int iu = (int)(rng_uniform(&rng) * g->nu);
            int iv = (int)(rng_uniform(&rng) * g->nv);
            v3 pix, dl, to_det;
            double dd2, cos_t, theta, p_dir, e_out, tau, x, mb[256];
            size_t pixel;
            if (iu > g->nu - 1)
                iu = g->nu - 1;
            if (iv > g->nv - 1)
                iv = g->nv - 1;
            pix = pixel_position(g, &c->fr, iu, iv);
            dl = vsub(pix, pos);
            dd2 = vdot(dl, dl);
            to_det = vdiv(dl, sqrt(dd2));
            cos_t = clampd(vdot(dir, to_det), -1.0, 1.0);
            theta = acos(cos_t);
            if (kind == K_COMPTON) {
                p_dir = p_lambda_compton(mat, energy, theta);
                e_out = energy * compton_energy_ratio(energy, theta);
            } else {
                p_dir = p_lambda_rayleigh(mat, energy, theta);
                e_out = energy;
            }
            mu_field(&c->scene, e_out, mb);
            ++h->rays;
            tau = trace_attenuation(ph, pos, to_det, mb, cfg->step_voxels, &h->sc_steps);
            x = pd_score(response_factor(c->resp, e_out), p_dir, w_split, n_pixels, dd2, tau);
            if (!isfinite(x))
                xo_throw(XS_E_RUNTIME,
                         "simulate_scatter: non-finite contribution (angle %d, bin %d, E %f "
                         "keV) - physics tables corrupt?",
                         c->angle_idx, bin, energy);
            pixel = (size_t)iv * g->nu + iu;
            hist_push(h, pixel, x);
            h->total += x;
        }
        if (kind == K_COMPTON) {
            double th, ap, phi;
            sample_compton(mat, energy, &rng, &th, &ap, &phi);
            dir = rotate_direction(dir, th, phi);
            energy = ap * XO_MEC2_KEV;
            mu_field(&c->scene, energy, ma);
        } else {
            double th, phi;
            sample_rayleigh(mat, energy, &rng, &th, &phi);
            dir = rotate_direction(dir, th, phi);
        }
        ++generation;
        if (generation >= cfg->max_interactions) {
            led_push(h, 3, weight);
            break;
        }
        if (w_min > 0.0 && weight < w_min) {
            if (rng_uniform(&rng) < cfg->roulette_survival) {
                const double boosted = weight / cfg->roulette_survival;
                led_push(h, 5, boosted - weight);
                weight = boosted;
            } else {
                led_push(h, 4, weight);
                break;
            }
        }
    }
}

/* ----- sink 1: REF's chunked fp64 accumulation (transport.cpp:256-322) */

typedef struct bin_stats {
    double sum_t, sum_t2;
    uint64_t n;
} bin_stats;

typedef struct ochunk {
    double* image;
    double* var_c;
    double* var_c2;
    oledger led;
    bin_stats* bins;
    int err_code;
    char err_msg[512];
} ochunk;

typedef struct pair_ent {
    size_t pixel;
    double x;
} pair_ent;

static int pair_cmp(const void* a, const void* b)
{
    const pair_ent* p = (const pair_ent*)a;
    const pair_ent* q = (const pair_ent*)b;
    if (p->pixel != q->pixel)
        return p->pixel < q->pixel ? -1 : 1;
    if (p->x != q->x)
        return p->x < q->x ? -1 : 1;
    return 0;
}

#define XO_CHUNKS 64

static void run_chunk(const octx* c, int chunk, ochunk* acc)
{
    ohist_out h;
    pair_ent* pairs = NULL;
    int pcap = 0;
    int bin;
    memset(&h, 0, sizeof h);
    for (bin = 0; bin < c->spec->n_bins; ++bin) {
        const uint64_t m = c->photons_per_bin[bin];
        uint64_t j, begin, end;
        if (m == 0)
            continue;
        begin = m * (uint64_t)chunk / XO_CHUNKS;
        end = m * (uint64_t)(chunk + 1) / XO_CHUNKS;
        for (j = begin; j < end; ++j) {
            int i;
            run_history(c, bin, j, &h);
            for (i = 0; i < h.n_scores; ++i)
                acc->image[h.pix[i]] += h.val[i];
            for (i = 0; i < h.n_led; ++i) {
                double* slot = &acc->led.initial + h.led_kind[i];
                *slot += h.led_val[i];
            }
            acc->bins[bin].sum_t += h.total;
            acc->bins[bin].sum_t2 += h.total * h.total;
            ++acc->bins[bin].n;
            if (c->cfg->track_variance && h.n_scores > 0) {
                size_t k = 0;
                if (h.n_scores > pcap) {
                    pcap = h.n_scores;
                    pairs = (pair_ent*)realloc(pairs, sizeof(pair_ent) * (size_t)pcap);
                }
                for (i = 0; i < h.n_scores; ++i) {
                    pairs[i].pixel = h.pix[i];
                    pairs[i].x = h.val[i];
                }
                qsort(pairs, (size_t)h.n_scores, sizeof(pair_ent), pair_cmp);
                while (k < (size_t)h.n_scores) {
                    const size_t pixel = pairs[k].pixel;
                    double cc = 0.0;
                    while (k < (size_t)h.n_scores && pairs[k].pixel == pixel)
                        cc += pairs[k++].x;
                    acc->var_c[pixel] += cc;
                    acc->var_c2[pixel] += cc * cc;
                }
            }
        }
    }
    free(pairs);
    free(h.pix);
    free(h.val);
}

typedef struct oworker {
    const octx* c;
    ochunk* chunks;
    int* next;
    pthread_mutex_t* mu;
} oworker;

static void* worker_main(void* arg) /* parallel_for (worker_pool.hpp:17-57) */
{
    oworker* w = (oworker*)arg;
    for (;;) {
        int chunk;
        xo_err e;
        pthread_mutex_lock(w->mu);
        chunk = (*w->next)++;
        pthread_mutex_unlock(w->mu);
        if (chunk >= XO_CHUNKS)
            break;
        tl_err = &e;
        if (setjmp(e.jb)) {
            w->chunks[chunk].err_code = e.code;
            snprintf(w->chunks[chunk].err_msg, sizeof w->chunks[chunk].err_msg, "%s", e.msg);
            tl_err = NULL;
            continue;
        }
        run_chunk(w->c, chunk, &w->chunks[chunk]);
        tl_err = NULL;
    }
    return NULL;
}

static void ctx_init(octx* c, const xs_phantom* ph, const xs_geometry* g, int angle_idx,
                     const xs_spectrum* spec, const xs_response* resp, const xs_sim_config* cfg,
                     const char* who)
{
    validate_sim_config(cfg);
    validate_spectrum(spec);
    validate_geometry(g);
    if (angle_idx < 0 || angle_idx >= g->n_angles)
        xo_throw(XS_E_OUT_OF_RANGE, "%s: angle index out of range", who);
    if (ph->n_materials > 256)
        xo_throw(XS_E_RUNTIME, "phantom: too many materials");
    c->ph = ph;
    c->g = g;
    c->angle_idx = angle_idx;
    c->fr = frame_of(g, angle_idx);
    c->spec = spec;
    c->resp = resp;
    c->cfg = cfg;
    c->photons_per_bin = (uint64_t*)calloc((size_t)spec->n_bins, sizeof(uint64_t));
    xo_apportion_photons(spec, cfg->photons_total, c->photons_per_bin);
    c->units = xs_accum_units_make(g, spec, c->photons_per_bin);
    scene_init(&c->scene, ph);
}

static void ctx_free(octx* c)
{
    free(c->photons_per_bin);
    scene_free(&c->scene);
}

int xo_simulate_scatter_stats(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                              const xs_spectrum* spec, const xs_response* resp,
                              const xs_sim_config* cfg, int32_t workers, xs_scatter_result* out)
{
    octx c;
    ochunk* chunks;
    size_t n_pix, i;
    int k, next = 0, nthreads;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    pthread_t* th;
    oworker wk;
    bin_stats* bins;
    double *var_c = NULL, *var_c2 = NULL, var_total;
    XO_TRY
    ctx_init(&c, ph, g, angle_idx, spec, resp, cfg, "simulate_scatter");
    XO_END
    n_pix = (size_t)g->nu * (size_t)g->nv;
    chunks = (ochunk*)calloc(XO_CHUNKS, sizeof(ochunk));
    for (k = 0; k < XO_CHUNKS; ++k) {
        chunks[k].image = (double*)calloc(n_pix, sizeof(double));
        chunks[k].bins = (bin_stats*)calloc((size_t)spec->n_bins, sizeof(bin_stats));
        if (cfg->track_variance) {
            chunks[k].var_c = (double*)calloc(n_pix, sizeof(double));
            chunks[k].var_c2 = (double*)calloc(n_pix, sizeof(double));
        }
    }
    nthreads = workers < 1 ? 1 : (workers > XO_CHUNKS ? XO_CHUNKS : workers);
    wk.c = &c;
    wk.chunks = chunks;
    wk.next = &next;
    wk.mu = &mu;
    th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (k = 0; k < nthreads; ++k)
        pthread_create(&th[k], NULL, worker_main, &wk);
    for (k = 0; k < nthreads; ++k)
        pthread_join(th[k], NULL);
    free(th);

    for (k = 0; k < XO_CHUNKS; ++k)
        if (chunks[k].err_code) {
            const int code = chunks[k].err_code;
            snprintf(tl_last, sizeof tl_last, "%s", chunks[k].err_msg);
            for (k = 0; k < XO_CHUNKS; ++k) {
                free(chunks[k].image);
                free(chunks[k].bins);
                free(chunks[k].var_c);
                free(chunks[k].var_c2);
            }
            free(chunks);
            ctx_free(&c);
            return code;
        }

    /* fixed-order chunk reduction (transport.cpp:282-304) */
    memset(out->image, 0, sizeof(double) * n_pix);
    memset(&out->ledger, 0, sizeof out->ledger);
    bins = (bin_stats*)calloc((size_t)spec->n_bins, sizeof(bin_stats));
    if (cfg->track_variance) {
        var_c = (double*)calloc(n_pix, sizeof(double));
        var_c2 = (double*)calloc(n_pix, sizeof(double));
    }
    for (k = 0; k < XO_CHUNKS; ++k) {
        const ochunk* a = &chunks[k];
        int b;
        for (i = 0; i < n_pix; ++i)
            out->image[i] += a->image[i];
        out->ledger.initial += a->led.initial;
        out->ledger.escaped += a->led.escaped;
        out->ledger.absorbed += a->led.absorbed;
        out->ledger.culled += a->led.culled;
        out->ledger.roulette_killed += a->led.killed;
        out->ledger.roulette_boost += a->led.boost;
        for (b = 0; b < spec->n_bins; ++b) {
            bins[b].sum_t += a->bins[b].sum_t;
            bins[b].sum_t2 += a->bins[b].sum_t2;
            bins[b].n += a->bins[b].n;
        }
        if (cfg->track_variance)
            for (i = 0; i < n_pix; ++i) {
                var_c[i] += a->var_c[i];
                var_c2[i] += a->var_c2[i];
            }
    }
    /* transport.cpp:306-322 */
    out->histories = 0;
    out->total = 0.0;
    var_total = 0.0;
    for (k = 0; k < spec->n_bins; ++k) {
        const bin_stats* bs = &bins[k];
        out->histories += bs->n;
        out->total += bs->sum_t;
        if (bs->n > 1) {
            const double s2 = (bs->sum_t2 - bs->sum_t * bs->sum_t / bs->n) / (bs->n - 1);
            var_total += bs->n * (s2 > 0.0 ? s2 : 0.0);
        }
    }
    out->total_std_error = sqrt(var_total);
    if (cfg->track_variance && out->variance) {
        const double n = (double)out->histories;
        const double den = n - 1.0 > 1.0 ? n - 1.0 : 1.0;
        for (i = 0; i < n_pix; ++i) {
            const double v = var_c2[i] - var_c[i] * var_c[i] / n;
            out->variance[i] = (v > 0.0 ? v : 0.0) * n / den;
        }
    }
    free(var_c);
    free(var_c2);
    free(bins);
    for (k = 0; k < XO_CHUNKS; ++k) {
        free(chunks[k].image);
        free(chunks[k].bins);
        free(chunks[k].var_c);
        free(chunks[k].var_c2);
    }
    free(chunks);
    ctx_free(&c);
    return XS_OK;
}

/* ----- sink 2: deterministic fixed-point accumulator (include/xscat_gpu.h) */

static void limb_add(uint64_t* slot, double x, int32_t log2_unit)
{
    uint64_t l[3];
    if (xs_quantize(ldexp(x, -log2_unit), l))
        xo_throw(XS_E_RUNTIME, "simulate_scatter: fixed-point tally overflow (value %g)", x);
    slot[0] += l[0];
    slot[1] += l[1];
    slot[2] += l[2];
}

int xo_scatter_accumulate_range(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                                const xs_spectrum* spec, const xs_response* resp,
                                const xs_sim_config* cfg, uint64_t hist_begin,
                                uint64_t hist_end, uint64_t* accum)
{
    octx c;
    ohist_out h;
    xs_accum_layout L;
    uint64_t base = 0;
    int bin;
    memset(&h, 0, sizeof h);
    XO_TRY
    ctx_init(&c, ph, g, angle_idx, spec, resp, cfg, "simulate_scatter");
    L = xs_accum_layout_make(g->nu, g->nv, spec->n_bins, cfg->track_variance);
    for (bin = 0; bin < spec->n_bins; ++bin) {
        const uint64_t m = c.photons_per_bin[bin];
        uint64_t lo = hist_begin > base ? hist_begin - base : 0;
        uint64_t hi = hist_end > base ? hist_end - base : 0;
        uint64_t j;
        if (hi > m)
            hi = m;
        for (j = lo; j < hi; ++j) {
            int i;
            uint64_t* bs = accum + L.off_bins + 8 * (uint64_t)bin;
            uint64_t* led = accum + L.off_ledger;
            run_history(&c, bin, j, &h);
            for (i = 0; i < h.n_scores; ++i)
                limb_add(accum + L.off_image + 4 * h.pix[i], h.val[i], c.units.log2_img);
            if (cfg->track_variance) {
                /* group this history's scores per pixel in production order */
                int a, b2;
                for (a = 0; a < h.n_scores; ++a) {
                    double cc;
                    int dup = 0;
                    for (b2 = 0; b2 < a; ++b2)
                        if (h.pix[b2] == h.pix[a]) {
                            dup = 1;
                            break;
                        }
                    if (dup)
                        continue;
                    cc = h.val[a];
                    for (b2 = a + 1; b2 < h.n_scores; ++b2)
                        if (h.pix[b2] == h.pix[a])
                            cc += h.val[b2];
                    limb_add(accum + L.off_variance + 4 * h.pix[a], cc * cc,
                             2 * c.units.log2_img);
                }
            }
            limb_add(bs, h.total, c.units.log2_img);
            limb_add(bs + 3, h.total * h.total, 2 * c.units.log2_img);
            for (i = 0; i < h.n_led; ++i)
                limb_add(led + 4 * h.led_kind[i], h.led_val[i], c.units.log2_w);
        }
        base += m;
    }
    accum[L.off_diag + 0] += h.fp_steps;
    accum[L.off_diag + 1] += h.sc_steps;
    accum[L.off_diag + 2] += hist_end > hist_begin ? hist_end - hist_begin : 0;
    accum[L.off_diag + 3] += h.rays;
    accum[L.off_diag + 4] += h.interactions;
    free(h.pix);
    free(h.val);
    ctx_free(&c);
    XO_END
    return XS_OK;
}

/* ----------------------------------------------------------------- primary
 * simulate_primary (transport.cpp:333-377) */

typedef struct oprim {
    const octx* c;
    double* image;
    const double* atten;
    const double* response;
    int* next_row;
    pthread_mutex_t* mu;
    int err_code;
    char err_msg[512];
} oprim;

static void* primary_worker(void* arg)
{
    oprim* p = (oprim*)arg;
    const octx* c = p->c;
    const xs_geometry* g = c->g;
    const int n_mats = c->ph->n_materials;
    const int n_bins = c->spec->n_bins;
    double* rho = (double*)malloc(sizeof(double) * (size_t)n_mats);
    xo_err e;
    tl_err = &e;
    if (setjmp(e.jb)) {
        p->err_code = e.code;
        snprintf(p->err_msg, sizeof p->err_msg, "%s", e.msg);
        tl_err = NULL;
        free(rho);
        return NULL;
    }
    for (;;) {
        int iv, iu;
        pthread_mutex_lock(p->mu);
        iv = (*p->next_row)++;
        pthread_mutex_unlock(p->mu);
        if (iv >= g->nv)
            break;
        for (iu = 0; iu < g->nu; ++iu) {
            const v3 pix = pixel_position(g, &c->fr, iu, iv);
            const v3 delta = vsub(pix, c->fr.src);
            const double d2 = vdot(delta, delta);
            const v3 rd = vdiv(delta, sqrt(d2));
            double value = 0.0;
            int b, m;
            trace_rho_lengths(c->ph, c->fr.src, rd, rho);
            for (b = 0; b < n_bins; ++b) {
                double tau = 0.0;
                for (m = 1; m < n_mats; ++m)
                    tau += p->atten[(size_t)b * n_mats + m] * rho[m];
                value += c->spec->weight[b] * p->response[b] * exp(-tau) / d2;
            }
            p->image[(size_t)iv * g->nu + iu] = value;
        }
    }
    tl_err = NULL;
    free(rho);
    return NULL;
}

int xo_simulate_primary(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                        const xs_spectrum* spec, const xs_response* resp,
                        const xs_sim_config* cfg, int32_t workers, double* image)
{
    octx c;
    double *atten, *response;
    int n_bins, n_mats, b, m, k, next = 0, nthreads, err = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    oprim* ps;
    pthread_t* th;
    XO_TRY
    ctx_init(&c, ph, g, angle_idx, spec, resp, cfg, "simulate_primary");
    n_bins = spec->n_bins;
    n_mats = ph->n_materials;
    atten = (double*)calloc((size_t)n_bins * n_mats, sizeof(double));
    response = (double*)calloc((size_t)n_bins, sizeof(double));
    for (b = 0; b < n_bins; ++b) {
        response[b] = response_factor(resp, spec->energy_kev[b]);
        for (m = 1; m < n_mats; ++m)
            if (c.scene.mats[m].has_tables)
                atten[(size_t)b * n_mats + m] = tab_loglog(&ph->materials[m].mu, spec->energy_kev[b]);
    }
    XO_END
    nthreads = workers < 1 ? 1 : workers;
    ps = (oprim*)calloc((size_t)nthreads, sizeof(oprim));
    th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (k = 0; k < nthreads; ++k) {
        ps[k].c = &c;
        ps[k].image = image;
        ps[k].atten = atten;
        ps[k].response = response;
        ps[k].next_row = &next;
        ps[k].mu = &mu;
        pthread_create(&th[k], NULL, primary_worker, &ps[k]);
    }
    for (k = 0; k < nthreads; ++k)
        pthread_join(th[k], NULL);
    for (k = 0; k < nthreads; ++k)
        if (ps[k].err_code && !err) {
            err = ps[k].err_code;
            snprintf(tl_last, sizeof tl_last, "%s", ps[k].err_msg);
        }
    free(th);
    free(ps);
    free(atten);
    free(response);
    ctx_free(&c);
    return err;
}

/* --------------------------------------------------------- post-processing
 * postprocess.cpp:11-271 */

int xo_sg_kernel(int32_t left, int32_t right, int32_t polyorder, double* kernel)
{
    const int n = left + right + 1;
    const int order = polyorder < n - 1 ? polyorder : n - 1;
    const int k = order + 1;
    double *xtx, *powers, *rhs, *coef;
    int j, m, a, b, col, r, c2;
    xtx = (double*)calloc((size_t)k * k, sizeof(double));
    powers = (double*)calloc((size_t)n * k, sizeof(double));
    rhs = (double*)calloc((size_t)k, sizeof(double));
    coef = (double*)calloc((size_t)k, sizeof(double));
    for (j = 0; j < n; ++j) {
        const double x = j - left;
        double p = 1.0;
        for (m = 0; m < k; ++m) {
            powers[(size_t)j * k + m] = p;
            p *= x;
        }
    }
    for (a = 0; a < k; ++a)
        for (b = 0; b < k; ++b) {
            double s = 0.0;
            for (j = 0; j < n; ++j)
                s += powers[(size_t)j * k + a] * powers[(size_t)j * k + b];
            xtx[(size_t)a * k + b] = s;
        }
    rhs[0] = 1.0;
    for (col = 0; col < k; ++col) {
        int pivot = col;
        double diag;
        for (r = col + 1; r < k; ++r)
            if (fabs(xtx[(size_t)r * k + col]) > fabs(xtx[(size_t)pivot * k + col]))
                pivot = r;
        if (pivot != col) {
            double t;
            for (c2 = 0; c2 < k; ++c2) {
                t = xtx[(size_t)col * k + c2];
                xtx[(size_t)col * k + c2] = xtx[(size_t)pivot * k + c2];
                xtx[(size_t)pivot * k + c2] = t;
            }
            t = rhs[col];
            rhs[col] = rhs[pivot];
            rhs[pivot] = t;
        }
        diag = xtx[(size_t)col * k + col];
        if (diag == 0.0) {
            snprintf(tl_last, sizeof tl_last, "sg_kernel: singular normal equations");
            free(xtx);
            free(powers);
            free(rhs);
            free(coef);
            return XS_E_RUNTIME;
        }
        for (r = col + 1; r < k; ++r) {
            const double f = xtx[(size_t)r * k + col] / diag;
            for (c2 = col; c2 < k; ++c2)
                xtx[(size_t)r * k + c2] -= f * xtx[(size_t)col * k + c2];
            rhs[r] -= f * rhs[col];
        }
    }
    for (r = k - 1; r >= 0; --r) {
        double s = rhs[r];
        for (c2 = r + 1; c2 < k; ++c2)
            s -= xtx[(size_t)r * k + c2] * coef[c2];
        coef[r] = s / xtx[(size_t)r * k + r];
    }
    for (j = 0; j < n; ++j) {
        double s = 0.0;
        for (m = 0; m < k; ++m)
            s += coef[m] * powers[(size_t)j * k + m];
        kernel[j] = s;
    }
    free(xtx);
    free(powers);
    free(rhs);
    free(coef);
    return XS_OK;
}

int xo_default_sg_spec(int32_t nu, int32_t nv, int32_t* window, int32_t* polyorder)
{
    const int smaller = nu < nv ? nu : nv;
    int w = (int)lround(15.0 * smaller / 576.0);
    w = (w | 1) > 5 ? (w | 1) : 5;
    {
        const int cap = smaller % 2 ? smaller : smaller - 1;
        w = w < cap ? w : cap;
    }
    *window = w;
    *polyorder = 3;
    return XS_OK;
}

static int validate_sg(int window, int polyorder)
{
    if (window < 5 || window % 2 == 0) {
        snprintf(tl_last, sizeof tl_last, "sg filter: window must be odd and >= 5");
        return XS_E_RUNTIME;
    }
    if (polyorder < 0 || polyorder >= window) {
        snprintf(tl_last, sizeof tl_last, "sg filter: polyorder must be < window");
        return XS_E_RUNTIME;
    }
    return XS_OK;
}

static void sg_pass(const double* in, double* out, int n, int stride, int half,
                    double* const* kernels)
{
    int i, j;
    for (i = 0; i < n; ++i) {
        const int left = i < half ? i : half;
        const int right = (n - 1 - i) < half ? (n - 1 - i) : half;
        const double* k = kernels[(size_t)left * (half + 1) + right];
        const double* base = in + (ptrdiff_t)(i - left) * stride;
        double s = 0.0;
        for (j = 0; j < left + right + 1; ++j)
            s += k[j] * base[(ptrdiff_t)j * stride];
        out[(ptrdiff_t)i * stride] = s;
    }
}

int xo_sg_smooth(const double* in, double* out, int32_t nu, int32_t nv, int32_t window,
                 int32_t polyorder)
{
    int half, l, r, iv, iu, st;
    double** kernels;
    double* tmp;
    if ((st = validate_sg(window, polyorder)))
        return st;
    if (nu < window || nv < window) {
        snprintf(tl_last, sizeof tl_last, "sg_smooth: image dims smaller than filter window");
        return XS_E_RUNTIME;
    }
    half = window / 2;
    kernels = (double**)calloc((size_t)(half + 1) * (half + 1), sizeof(double*));
    for (l = 0; l <= half; ++l)
        for (r = 0; r <= half; ++r) {
            double* k = (double*)malloc(sizeof(double) * (size_t)(l + r + 1));
            xo_sg_kernel(l, r, polyorder, k);
            kernels[(size_t)l * (half + 1) + r] = k;
        }
    tmp = (double*)calloc((size_t)nu * nv, sizeof(double));
    for (iv = 0; iv < nv; ++iv)
        sg_pass(in + (size_t)iv * nu, tmp + (size_t)iv * nu, nu, 1, half, kernels);
    for (iu = 0; iu < nu; ++iu)
        sg_pass(tmp + iu, out + iu, nv, nu, half, kernels);
    for (l = 0; l < (half + 1) * (half + 1); ++l)
        free(kernels[l]);
    free(kernels);
    free(tmp);
    return XS_OK;
}

int xo_interpolate_angles(const double* in, const double* src, int32_t n_src, double* out,
                          const double* tgt, int32_t n_tgt, int32_t nu, int32_t nv)
{
    const double period = 2.0 * XO_PI;
    const size_t np = (size_t)nu * nv;
    int i, t;
    for (i = 1; i < n_src; ++i)
        if (!(src[i] > src[i - 1])) {
            snprintf(tl_last, sizeof tl_last, "interpolate_angles: source angles not sorted");
            return XS_E_RUNTIME;
        }
    for (i = 1; i < n_tgt; ++i)
        if (!(tgt[i] > tgt[i - 1])) {
            snprintf(tl_last, sizeof tl_last, "interpolate_angles: target angles not sorted");
            return XS_E_RUNTIME;
        }
    for (t = 0; t < n_tgt; ++t) {
        const double b = tgt[t];
        int hi = 0, lo;
        double a_lo, a_hi, w;
        size_t p;
        while (hi < n_src && src[hi] < b) /* lower_bound */
            ++hi;
        if (hi < n_src && src[hi] == b) {
            memcpy(out + (size_t)t * np, in + (size_t)hi * np, sizeof(double) * np);
            continue;
        }
        if (n_src < 2) {
            snprintf(tl_last, sizeof tl_last, "interpolate_angles: missing bracket for angle %f",
                     b);
            return XS_E_RUNTIME;
        }
        if (hi == 0) {
            lo = n_src - 1;
            a_lo = src[lo] - period;
            a_hi = src[0];
        } else if (hi == n_src) {
            lo = n_src - 1;
            hi = 0;
            a_lo = src[lo];
            a_hi = src[0] + period;
        } else {
            lo = hi - 1;
            a_lo = src[lo];
            a_hi = src[hi];
        }
        w = (b - a_lo) / (a_hi - a_lo);
        for (p = 0; p < np; ++p)
            out[(size_t)t * np + p] =
                (1.0 - w) * in[(size_t)lo * np + p] + w * in[(size_t)hi * np + p];
    }
    return XS_OK;
}

static double cr_fetch(const double* line, int n, int stride, int i) /* :201-212 */
{
    if (n == 1)
        return line[0];
    if (i < 0)
        return line[0] + i * (line[stride] - line[0]);
    if (i >= n)
        return line[(ptrdiff_t)(n - 1) * stride] +
               (i - (n - 1)) *
                   (line[(ptrdiff_t)(n - 1) * stride] - line[(ptrdiff_t)(n - 2) * stride]);
    return line[(ptrdiff_t)i * stride];
}

static void cr_pass(const double* in, double* out, int n_in, int n_out, int s_in, int s_out)
{
    const double scale = (double)n_in / n_out;
    int i;
    for (i = 0; i < n_out; ++i) {
        const double x = (i + 0.5) * scale - 0.5;
        const int base = (int)floor(x);
        const double t = x - base;
        const double t2 = t * t, t3 = t2 * t;
        const double w0 = 0.5 * (-t3 + 2.0 * t2 - t);
        const double w1 = 0.5 * (3.0 * t3 - 5.0 * t2 + 2.0);
        const double w2 = 0.5 * (-3.0 * t3 + 4.0 * t2 + t);
        const double w3 = 0.5 * (t3 - t2);
        out[(ptrdiff_t)i * s_out] =
            w0 * cr_fetch(in, n_in, s_in, base - 1) + w1 * cr_fetch(in, n_in, s_in, base) +
            w2 * cr_fetch(in, n_in, s_in, base + 1) + w3 * cr_fetch(in, n_in, s_in, base + 2);
    }
}

int xo_upsample_image(const double* in, int32_t nu, int32_t nv, double* out, int32_t nu_out,
                      int32_t nv_out)
{
    double* tmp;
    int iv, iu;
    if (nu_out < nu || nv_out < nv) {
        snprintf(tl_last, sizeof tl_last, "upsample_image: target dims must be >= source dims");
        return XS_E_RUNTIME;
    }
    if (nu < 1 || nv < 1) {
        snprintf(tl_last, sizeof tl_last, "upsample_image: degenerate source");
        return XS_E_RUNTIME;
    }
    tmp = (double*)calloc((size_t)nu_out * nv, sizeof(double));
    for (iv = 0; iv < nv; ++iv)
        cr_pass(in + (size_t)iv * nu, tmp + (size_t)iv * nu_out, nu, nu_out, 1, 1);
    for (iu = 0; iu < nu_out; ++iu)
        cr_pass(tmp + iu, out + iu, nv, nv_out, nu_out, nu_out);
    free(tmp);
    return XS_OK;
}

int xo_downsample_average(const double* in, int32_t nu, int32_t nv, double* out,
                          int32_t nu_out, int32_t nv_out)
{
    int ov, ou, v, u;
    if (nu_out > nu || nv_out > nv || nu_out < 1 || nv_out < 1) {
        snprintf(tl_last, sizeof tl_last, "downsample_average: bad target dims");
        return XS_E_RUNTIME;
    }
    for (ov = 0; ov < nv_out; ++ov) {
        const int v0 = ov * nv / nv_out, v1 = (ov + 1) * nv / nv_out;
        for (ou = 0; ou < nu_out; ++ou) {
            const int u0 = ou * nu / nu_out, u1 = (ou + 1) * nu / nu_out;
            double s = 0.0;
            for (v = v0; v < v1; ++v)
                for (u = u0; u < u1; ++u)
                    s += in[(size_t)v * nu + u];
            out[(size_t)ov * nu_out + ou] = s / ((v1 - v0) * (u1 - u0));
        }
    }
    return XS_OK;
}

/* ------------------------------------------------ correction-loop stages */

/* REF intensity_to_attenuation (recon.cpp:324-348). */
int xo_intensity_to_attenuation(const double* intensity, const double* flat, int32_t nu, int32_t nv,
                                int32_t n, double* out)
{
    const size_t np = (size_t)nu * nv;
    size_t bad = 0, p;
    int i;
    for (p = 0; p < np; ++p)
        if (!(flat[p] > 0.0))
            ++bad;
    for (i = 0; i < n; ++i)
        for (p = 0; p < np; ++p) {
            const double v = intensity[(size_t)i * np + p];
            if (!(v > 0.0)) {
                ++bad;
                out[(size_t)i * np + p] = 0.0;
                continue;
            }
            out[(size_t)i * np + p] = log(flat[p] / v);
        }
    if (bad > 0) {
        snprintf(tl_last, sizeof tl_last,
                 "intensity_to_attenuation: %zu non-positive pixels (underexposed or invalid data)", bad);
        return XS_E_RUNTIME;
    }
    return XS_OK;
}

/* REF correct_projections (correction.cpp:58-86), Eq. 8. */
int xo_correct_projections(const double* a, const double* primary, const double* scatter, int32_t nu,
                           int32_t nv, int32_t n, double* out, uint64_t* clamped)
{
    const size_t total = (size_t)nu * nv * n;
    size_t k, cl = 0;
    for (k = 0; k < total; ++k) {
        double is = scatter[k];
        if (!(primary[k] > 0.0)) {
            snprintf(tl_last, sizeof tl_last, "correct_projections: non-positive primary pixel");
            return XS_E_RUNTIME;
        }
        if (is < 0.0) {
            is = 0.0;
            ++cl;
        }
        out[k] = a[k] - log(primary[k] / (primary[k] + is));
    }
    *clamped = cl;
    return XS_OK;
}

/* REF correction.cpp:199-246, the loop's tail after the Monte Carlo runs:
 * SG per scatter image, angle interpolation, up-sampling of both stacks,
 * primary floor at 1e-12 of each view's peak, mean scatter fraction, Eq. 8. */
int xo_correction_tail(const double* scatter_sub, const double* sub_angles, int32_t n_sub,
                       const double* primary_mc, const double* full_angles, int32_t n_full, int32_t nu,
                       int32_t nv, int32_t sg_window, int32_t sg_order, const double* a, int32_t nu_out,
                       int32_t nv_out, double* corrected, double* mean_fraction, uint64_t* clamped)
{
    const size_t np = (size_t)nu * nv, npo = (size_t)nu_out * nv_out;
    double *sg = (double*)malloc(np * (n_sub ? n_sub : 1) * sizeof(double));
    double *full = (double*)malloc(np * (n_full ? n_full : 1) * sizeof(double));
    double *s_hi = (double*)malloc(npo * (n_full ? n_full : 1) * sizeof(double));
    double *p_hi = (double*)malloc(npo * (n_full ? n_full : 1) * sizeof(double));
    double frac_sum = 0.0;
    size_t frac_n = 0, p;
    int i, rc = XS_OK;
    for (i = 0; i < n_sub && rc == XS_OK; ++i)
        rc = xo_sg_smooth(scatter_sub + i * np, sg + i * np, nu, nv, sg_window, sg_order);
    if (rc == XS_OK)
        rc = xo_interpolate_angles(sg, sub_angles, n_sub, full, full_angles, n_full, nu, nv);
    for (i = 0; i < n_full && rc == XS_OK; ++i) {
        rc = xo_upsample_image(full + i * np, nu, nv, s_hi + i * npo, nu_out, nv_out);
        if (rc == XS_OK)
            rc = xo_upsample_image(primary_mc + i * np, nu, nv, p_hi + i * npo, nu_out, nv_out);
    }
    for (i = 0; i < n_full && rc == XS_OK; ++i) { /* correction.cpp:212-221 */
        double peak = 0.0, floor_val;
        double* img = p_hi + i * npo;
        for (p = 0; p < npo; ++p)
            peak = img[p] > peak ? img[p] : peak;
        floor_val = 1e-12 * peak;
        for (p = 0; p < npo; ++p)
            img[p] = img[p] > floor_val ? img[p] : floor_val;
    }
    if (rc == XS_OK) { /* correction.cpp:226-239 */
        for (p = 0; p < npo * n_full; ++p) {
            const double is = s_hi[p] > 0.0 ? s_hi[p] : 0.0;
            if (p_hi[p] + is > 0.0) {
                frac_sum += is / (p_hi[p] + is);
                ++frac_n;
            }
        }
        *mean_fraction = frac_n ? frac_sum / frac_n : 0.0;
        rc = xo_correct_projections(a, p_hi, s_hi, nu_out, nv_out, n_full, corrected, clamped);
    }
    free(sg);
    free(full);
    free(s_hi);
    free(p_hi);
    return rc;
}

/* ------------------------------------------------------------------ FDK */
/* REF fbp_reconstruct (recon.cpp:58-157): cosine weighting, direct row
 * convolution with the ramp kernel (recon.cpp:23-43), distance-weighted
 * bilinear backprojection accumulated in float in view order, x 100. */
static double xo_ramlak(int k, double du)
{
    const double pi = 3.14159265358979323846;
    if (k == 0)
        return 1.0 / (8.0 * du * du);
    if (k % 2 == 0)
        return 0.0;
    return -1.0 / (2.0 * pi * pi * k * k * du * du);
}

int xo_fbp_reconstruct(const double* stack, const double* angles, int32_t n_views, int32_t nu, int32_t nv,
                       const xs_geometry* g, const int32_t dims[3], const double voxel[3], int32_t hann,
                       float* volume)
{
    const double pi = 3.14159265358979323846;
    const double fan = 2.0 * atan(0.5 * g->nu * g->pixel_pitch / g->sdd);
    double span = 0.0, R, D, du, dv, x0, y0, z0;
    double *kern, *dbeta, *q, *w;
    size_t np = (size_t)nu * nv, nvox = (size_t)dims[0] * dims[1] * dims[2], p;
    int i, k, iv, iu, j, view, ix, iy, iz;
    if (n_views <= 0) {
        snprintf(tl_last, sizeof tl_last, "fbp: empty projection stack");
        return XS_E_RUNTIME;
    }
    if (n_views >= 2) {
        double max_gap = 2.0 * pi + angles[0] - angles[n_views - 1];
        for (i = 1; i < n_views; ++i)
            if (angles[i] - angles[i - 1] > max_gap)
                max_gap = angles[i] - angles[i - 1];
        span = 2.0 * pi - max_gap;
    }
    if (n_views < 2 || span + 1e-9 < pi + fan) {
        snprintf(tl_last, sizeof tl_last, "fbp: insufficient angular coverage (need >= 180 deg + fan)");
        return XS_E_RUNTIME;
    }
    R = g->sod;
    D = g->sdd;
    du = g->pixel_pitch * R / D;
    dv = du;
    dbeta = (double*)malloc(sizeof(double) * n_views);
    for (i = 0; i < n_views; ++i) {
        const double prev = (i == 0) ? angles[n_views - 1] - 2.0 * pi : angles[i - 1];
        const double next = (i == n_views - 1) ? angles[0] + 2.0 * pi : angles[i + 1];
        dbeta[i] = 0.5 * (next - prev);
    }
    kern = (double*)malloc(sizeof(double) * (2 * (size_t)nu - 1));
    for (k = -(nu - 1); k <= nu - 1; ++k) {
        double v = xo_ramlak(k, du);
        if (hann)
            v = 0.5 * xo_ramlak(k, du) + 0.25 * (xo_ramlak(k - 1, du) + xo_ramlak(k + 1, du));
        kern[k + nu - 1] = v;
    }
    q = (double*)malloc(sizeof(double) * np * n_views);
    w = (double*)malloc(sizeof(double) * np);
    for (view = 0; view < n_views; ++view) {
        const double* img = stack + (size_t)view * np;
        for (iv = 0; iv < nv; ++iv) {
            const double vv = (iv + 0.5 - 0.5 * nv) * dv;
            for (iu = 0; iu < nu; ++iu) {
                const double uu = (iu + 0.5 - 0.5 * nu) * du;
                w[(size_t)iv * nu + iu] = img[(size_t)iv * nu + iu] * R / sqrt(R * R + uu * uu + vv * vv);
            }
        }
        for (iv = 0; iv < nv; ++iv) {
            const double* row = w + (size_t)iv * nu;
            double* out = q + (size_t)view * np + (size_t)iv * nu;
            for (i = 0; i < nu; ++i) {
                double s = 0.0;
                for (j = 0; j < nu; ++j)
                    s += row[j] * kern[i - j + nu - 1];
                out[i] = s * du;
            }
        }
    }
    for (p = 0; p < nvox; ++p)
        volume[p] = 0.0f;
    x0 = -0.5 * dims[0] * voxel[0];
    y0 = -0.5 * dims[1] * voxel[1];
    z0 = -0.5 * dims[2] * voxel[2];
    for (iz = 0; iz < dims[2]; ++iz) {
        const double z = z0 + (iz + 0.5) * voxel[2];
        for (view = 0; view < n_views; ++view) {
            const double beta = angles[view];
            const double cb = cos(beta), sb = sin(beta);
            const double* qv = q + (size_t)view * np;
            for (iy = 0; iy < dims[1]; ++iy) {
                const double y = y0 + (iy + 0.5) * voxel[1];
                for (ix = 0; ix < dims[0]; ++ix) {
                    const double x = x0 + (ix + 0.5) * voxel[0];
                    const double s_comp = x * cb + y * sb;
                    const double t_comp = -x * sb + y * cb;
                    const double L = R - s_comp;
                    double pu, pv, fu, fv, val;
                    int u0, v0;
                    if (L <= 1e-9)
                        continue;
                    pu = (R * t_comp / L) / du + 0.5 * nu - 0.5;
                    pv = (R * z / L) / dv + 0.5 * nv - 0.5;
                    if (pu < 0.0 || pu > nu - 1 || pv < 0.0 || pv > nv - 1)
                        continue;
                    u0 = (int)pu < nu - 2 ? (int)pu : nu - 2;
                    v0 = (int)pv < nv - 2 ? (int)pv : nv - 2;
                    fu = pu - u0;
                    fv = pv - v0;
                    val = (1 - fu) * (1 - fv) * qv[(size_t)v0 * nu + u0] + fu * (1 - fv) * qv[(size_t)v0 * nu + u0 + 1] +
                          (1 - fu) * fv * qv[(size_t)(v0 + 1) * nu + u0] + fu * fv * qv[(size_t)(v0 + 1) * nu + u0 + 1];
                    volume[(size_t)ix + (size_t)dims[0] * ((size_t)iy + (size_t)dims[1] * iz)] +=
                        (float)(dbeta[view] * R * R / (L * L) * val);
                }
            }
        }
    }
    for (p = 0; p < nvox; ++p)
        volume[p] *= 100.0f;
    free(dbeta);
    free(kern);
    free(q);
    free(w);
    return XS_OK;
}


/* ---------------------------------------------------------- segmentation
 * recon.cpp:159-322. */

/* recon.cpp:159-240 */
int xo_otsu_thresholds(const float* vol, const int32_t dims[3], int32_t n_classes, int32_t bins,
                       double* thresholds)
{
    const int mx = dims[0] / 20 > 0 ? dims[0] / 20 : 0, my = dims[1] / 20 > 0 ? dims[1] / 20 : 0,
              mz = dims[2] / 20 > 0 ? dims[2] / 20 : 0;
    double lo = INFINITY, hi = -INFINITY, scale, *count, *pc, *ps, *best;
    int *arg, ix, iy, iz, b, k, m, cuts[4], W = bins + 1;
    const double neg_inf = -INFINITY;
    if (n_classes < 2 || n_classes > 4) {
        snprintf(tl_last, sizeof tl_last, "otsu: n_classes must be in [2,4]");
        return XS_E_INVALID_ARGUMENT;
    }
    if (bins < n_classes) {
        snprintf(tl_last, sizeof tl_last, "otsu: too few histogram bins");
        return XS_E_INVALID_ARGUMENT;
    }
#define XO_AT(x, y, z) vol[(size_t)(x) + (size_t)dims[0] * ((size_t)(y) + (size_t)dims[1] * (size_t)(z))]
    for (iz = mz; iz < dims[2] - mz; ++iz)
        for (iy = my; iy < dims[1] - my; ++iy)
            for (ix = mx; ix < dims[0] - mx; ++ix) {
                const double v = XO_AT(ix, iy, iz);
                lo = (v < lo) ? v : lo; /* std::min(lo, v) */
                hi = (hi < v) ? v : hi; /* std::max(hi, v) */
            }
    if (!(hi > lo)) {
        snprintf(tl_last, sizeof tl_last, "otsu: degenerate histogram");
        return XS_E_RUNTIME;
    }
    count = (double*)calloc((size_t)bins, sizeof(double));
    scale = bins / (hi - lo);
    for (iz = mz; iz < dims[2] - mz; ++iz)
        for (iy = my; iy < dims[1] - my; ++iy)
            for (ix = mx; ix < dims[0] - mx; ++ix) {
                const double t = (XO_AT(ix, iy, iz) - lo) * scale;
                /* static_cast<int>; out-of-range / NaN convert to INT_MIN on x86-64 */
                b = (t == t && t > -2147483649.0 && t < 2147483648.0) ? (int)t : (-2147483647 - 1);
                b = b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
                count[b] += 1.0;
            }
#undef XO_AT
    pc = (double*)calloc((size_t)W, sizeof(double));
    ps = (double*)calloc((size_t)W, sizeof(double));
    for (b = 0; b < bins; ++b) {
        pc[b + 1] = pc[b] + count[b];
        ps[b + 1] = ps[b] + count[b] * (b + 0.5);
    }
    best = (double*)malloc(sizeof(double) * (size_t)(n_classes + 1) * W);
    arg = (int*)malloc(sizeof(int) * (size_t)(n_classes + 1) * W);
    for (b = 0; b < (n_classes + 1) * W; ++b) {
        best[b] = neg_inf;
        arg[b] = -1;
    }
    best[0] = 0.0;
    for (k = 1; k <= n_classes; ++k)
        for (b = k; b <= bins; ++b)
            for (m = k - 1; m < b; ++m) {
                double sc, cand, n;
                if (best[(k - 1) * W + m] == neg_inf)
                    continue;
                n = pc[b] - pc[m];
                if (n <= 0.0) {
                    sc = neg_inf;
                } else {
                    const double s = ps[b] - ps[m];
                    sc = s * s / n;
                }
                cand = best[(k - 1) * W + m] + sc;
                if (cand > best[k * W + b]) {
                    best[k * W + b] = cand;
                    arg[k * W + b] = m;
                }
            }
    if (best[n_classes * W + bins] == neg_inf) {
        free(count), free(pc), free(ps), free(best), free(arg);
        snprintf(tl_last, sizeof tl_last, "otsu: degenerate histogram");
        return XS_E_RUNTIME;
    }
    /* backtrack; the cuts come out descending, the last one (0) is dropped */
    b = bins;
    for (k = n_classes; k >= 1; --k) {
        cuts[k - 1] = arg[k * W + b];
        b = arg[k * W + b];
    }
    for (k = 1; k < n_classes; ++k)
        thresholds[k - 1] = lo + cuts[k] / scale;
    free(count), free(pc), free(ps), free(best), free(arg);
    return XS_OK;
}

/* recon.cpp:242-262 */
int xo_segment_volume(const float* vol, uint64_t n, const double* thr, int32_t n_thr, int32_t n_class_map,
                      uint8_t* labels)
{
    uint64_t i;
    int t;
    for (t = 1; t < n_thr; ++t)
        if (!(thr[t] > thr[t - 1])) {
            snprintf(tl_last, sizeof tl_last, "segment_volume: thresholds must be strictly increasing");
            return XS_E_RUNTIME;
        }
    if (n_class_map != n_thr + 1) {
        snprintf(tl_last, sizeof tl_last, "segment_volume: class_map must cover all %d classes", n_thr + 1);
        return XS_E_RUNTIME;
    }
    for (i = 0; i < n; ++i) {
        const double v = vol[i];
        uint8_t label = 0;
        while (label < n_thr && v >= thr[label])
            ++label;
        labels[i] = label;
    }
    return XS_OK;
}

/* recon.cpp:264-322, then validate_phantom (phantom.cpp:33-56) */
int xo_to_density_phantom(const uint8_t* labels, const int32_t src[3], const xs_class_spec* cls,
                          int32_t n_classes, const int32_t tgt[3], int32_t n_materials,
                          const xs_material* materials, uint8_t* ids, float* dens)
{
    const uint64_t n_src = (uint64_t)src[0] * src[1] * src[2];
    uint64_t i, votes[256];
    int ox, oy, oz, ix, iy, iz, l;
    for (i = 0; i < n_src; ++i)
        if (labels[i] >= n_classes) {
            snprintf(tl_last, sizeof tl_last, "to_density_phantom: unmapped label %d", (int)labels[i]);
            return XS_E_RUNTIME;
        }
    for (oz = 0; oz < tgt[2]; ++oz) {
        const int z0 = oz * src[2] / tgt[2], z1 = (oz + 1) * src[2] / tgt[2];
        for (oy = 0; oy < tgt[1]; ++oy) {
            const int y0 = oy * src[1] / tgt[1], y1 = (oy + 1) * src[1] / tgt[1];
            for (ox = 0; ox < tgt[0]; ++ox) {
                const int x0 = ox * src[0] / tgt[0], x1 = (ox + 1) * src[0] / tgt[0];
                const size_t cell = (size_t)ox + (size_t)tgt[0] * ((size_t)oy + (size_t)tgt[1] * oz);
                double rho_sum = 0.0;
                uint64_t cnt = 0;
                int mode = 0;
                for (l = 0; l < n_classes; ++l)
                    votes[l] = 0;
                for (iz = z0; iz < z1; ++iz)
                    for (iy = y0; iy < y1; ++iy)
                        for (ix = x0; ix < x1; ++ix) {
                            const uint8_t label =
                                labels[(size_t)ix + (size_t)src[0] * ((size_t)iy + (size_t)src[1] * iz)];
                            ++votes[label];
                            rho_sum += cls[label].density;
                            ++cnt;
                        }
                for (l = 1; l < n_classes; ++l)
                    if (votes[l] >= votes[mode])
                        mode = l;
                if (cls[mode].material_id == 0) {
                    ids[cell] = 0;
                    dens[cell] = 0.0f;
                } else {
                    ids[cell] = (uint8_t)cls[mode].material_id;
                    dens[cell] = (float)(rho_sum / (double)cnt);
                }
            }
        }
    }
    if (materials) {
        const uint64_t n_out = (uint64_t)tgt[0] * tgt[1] * tgt[2];
        for (i = 0; i < n_out; ++i) {
            const int id = ids[i];
            if (id >= n_materials) {
                snprintf(tl_last, sizeof tl_last, "phantom: material id %d has no loaded material", id);
                return XS_E_RUNTIME;
            }
            if (id != 0 && materials[id].mu.n <= 0) {
                snprintf(tl_last, sizeof tl_last, "phantom: material id %d (%s) has no tables", id,
                         materials[id].name ? materials[id].name : "?");
                return XS_E_RUNTIME;
            }
            if (!(dens[i] >= 0.0f)) {
                snprintf(tl_last, sizeof tl_last, "phantom: negative density");
                return XS_E_RUNTIME;
            }
            if (id == 0 && dens[i] != 0.0f) {
                snprintf(tl_last, sizeof tl_last, "phantom: vacuum voxel with nonzero density");
                return XS_E_RUNTIME;
            }
        }
    }
    return XS_OK;
}
