/*
 * oracle.c -- CPU restatement of the reference (maniplan) hot path, FP64.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Not part of the product path.
 *
 * Each function names the reference function it restates
 * (paths relative to /root/reference/pkg/src/maniplan/).  The arithmetic
 * grouping follows the reference statement by statement because the test
 * suite pins this file bit-exactly against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py); numpy reductions are
 * reproduced with numpy's pairwise summation order (orc_np_sum).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fno-builtin-sin
 * -fno-builtin-cos, the reference's flags from pkg/setup.py:45-53).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MAXN 32   /* joints */
#define MAXM 5    /* error rows: _compiled.pyx:25-27 MAX_ERR */

/* ------------------------------------------------------------------ */
/* numpy reductions                                                    */
/* ------------------------------------------------------------------ */

/* numpy's pairwise summation (umath loops_utils: pairwise_sum) for the
 * contiguous reductions `(d*d).sum()` used by nearest/steer/connect/gaps
 * (planner.py:200-201,208,371,398; projection.py:133-134). */
double orc_np_sum(const double *a, int n)
{
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        int i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) +
                     ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return orc_np_sum(a, n2) + orc_np_sum(a + n2, n - n2);
}

static double sqnorm_diff_np(const double *a, const double *b, int n)
{
    double d[MAXN];
    for (int k = 0; k < n; k++) {
        double t = a[k] - b[k];
        d[k] = t * t;
    }
    return orc_np_sum(d, n);
}

/* ------------------------------------------------------------------ */
/* primitive clearances (pure.py:40-69)                                */
/* ------------------------------------------------------------------ */

static double axis_gap_sq(double c, double lo, double hi, double acc)
{
    if (c < lo) {
        double t = lo - c;
        return acc + t * t;
    }
    if (c > hi) {
        double t = c - hi;
        return acc + t * t;
    }
    return acc;
}

double orc_sphere_aabb_clearance(double cx, double cy, double cz, double r,
                                 double lx, double ly, double lz,
                                 double hx, double hy, double hz)
{
    double d2 = 0.0;
    d2 = axis_gap_sq(cx, lx, hx, d2);
    d2 = axis_gap_sq(cy, ly, hy, d2);
    d2 = axis_gap_sq(cz, lz, hz, d2);
    return sqrt(d2) - r;
}

double orc_sphere_sphere_clearance(double ax, double ay, double az, double ar,
                                   double bx, double by, double bz, double br)
{
    double dx = ax - bx, dy = ay - by, dz = az - bz;
    /* -(ar+br) keeps the value symmetric (pure.py:67-69) */
    return sqrt((dx * dx + dy * dy) + dz * dz) - (ar + br);
}

/* ------------------------------------------------------------------ */
/* 3x3 algebra (pure.py:76-177)                                        */
/* ------------------------------------------------------------------ */

static void m3mul(const double *a, const double *b, double *o)
{
    double t[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++)
            t[3 * i + j] = (a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j]) +
                           a[3 * i + 2] * b[6 + j];
    memcpy(o, t, sizeof t);
}

static void m3vec(const double *a, double x, double y, double z, double *o)
{
    double t0 = (a[0] * x + a[1] * y) + a[2] * z;
    double t1 = (a[3] * x + a[4] * y) + a[5] * z;
    double t2 = (a[6] * x + a[7] * y) + a[8] * z;
    o[0] = t0;
    o[1] = t1;
    o[2] = t2;
}

/* Rodrigues rotation about a unit axis (pure.py:101-118) */
static void axis_angle(double x, double y, double z, double ang, double *o)
{
    double c = cos(ang);
    double s = sin(ang);
    double t = 1.0 - c;
    double tx = t * x, ty = t * y, tz = t * z;
    double sx = s * x, sy = s * y, sz = s * z;
    double txy = tx * y, txz = tx * z, tyz = ty * z;
    o[0] = tx * x + c; o[1] = txy - sz;     o[2] = txz + sy;
    o[3] = txy + sz;   o[4] = ty * y + c;   o[5] = tyz - sx;
    o[6] = txz - sy;   o[7] = tyz + sx;     o[8] = tz * z + c;
}

static void qmul(double aw, double ax, double ay, double az,
                 double bw, double bx, double by, double bz, double *o)
{
    o[0] = ((aw * bw - ax * bx) - ay * by) - az * bz;
    o[1] = ((aw * bx + ax * bw) + ay * bz) - az * by;
    o[2] = ((aw * by - ax * bz) + ay * bw) + az * bx;
    o[3] = ((aw * bz + ax * by) - ay * bx) + az * bw;
}

/* rotation -> unit quaternion, w >= 0 (pure.py:130-159) */
static void quat_of(const double *r, double *q)
{
    double w, x, y, z, s;
    double tr = (r[0] + r[4]) + r[8];
    if (tr > 0.0) {
        s = sqrt(tr + 1.0) * 2.0;
        w = 0.25 * s;
        x = (r[7] - r[5]) / s;
        y = (r[2] - r[6]) / s;
        z = (r[3] - r[1]) / s;
    } else if (r[0] > r[4] && r[0] > r[8]) {
        s = sqrt(((1.0 + r[0]) - r[4]) - r[8]) * 2.0;
        w = (r[7] - r[5]) / s;
        x = 0.25 * s;
        y = (r[1] + r[3]) / s;
        z = (r[2] + r[6]) / s;
    } else if (r[4] > r[8]) {
        s = sqrt(((1.0 + r[4]) - r[0]) - r[8]) * 2.0;
        w = (r[2] - r[6]) / s;
        x = (r[1] + r[3]) / s;
        y = 0.25 * s;
        z = (r[5] + r[7]) / s;
    } else {
        s = sqrt(((1.0 + r[8]) - r[0]) - r[4]) * 2.0;
        w = (r[3] - r[1]) / s;
        x = (r[2] + r[6]) / s;
        y = (r[5] + r[7]) / s;
        z = 0.25 * s;
    }
    if (w < 0.0) {
        w = -w; x = -x; y = -y; z = -z;
    }
    q[0] = w; q[1] = x; q[2] = y; q[3] = z;
}

void orc_rot_from_quat(double w, double x, double y, double z, double *o)
{
    /* pure.py:162-177 (packing helper) */
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, xz = x * z, yz = y * z;
    double wx = w * x, wy = w * y, wz = w * z;
    o[0] = 1.0 - 2.0 * (yy + zz); o[1] = 2.0 * (xy - wz); o[2] = 2.0 * (xz + wy);
    o[3] = 2.0 * (xy + wz); o[4] = 1.0 - 2.0 * (xx + zz); o[5] = 2.0 * (yz - wx);
    o[6] = 2.0 * (xz - wy); o[7] = 2.0 * (yz + wx); o[8] = 1.0 - 2.0 * (xx + yy);
}

/* ------------------------------------------------------------------ */
/* forward kinematics (pure.py:188-248)                                */
/* ------------------------------------------------------------------ */

typedef struct {
    double R[MAXN][9];
    double p[MAXN][3];
    double axis_w[MAXN][3];
    double org_w[MAXN][3];
} chain_t;

static void fk_chain(const orc_robot *rb, const double *q, chain_t *c)
{
    double pr[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double px = 0.0, py = 0.0, pz = 0.0;
    for (int i = 0; i < rb->n; i++) {
        double r1[9], t[3], aw[3];
        m3mul(pr, rb->origin_r + 9 * i, r1);
        const double *o = rb->origin_p + 3 * i;
        m3vec(pr, o[0], o[1], o[2], t);
        double p1x = t[0] + px, p1y = t[1] + py, p1z = t[2] + pz;
        const double *ax = rb->axes + 3 * i;
        m3vec(r1, ax[0], ax[1], ax[2], aw);
        memcpy(c->axis_w[i], aw, sizeof aw);
        c->org_w[i][0] = p1x; c->org_w[i][1] = p1y; c->org_w[i][2] = p1z;
        if (rb->jtypes[i] == 0) {
            double rot[9];
            axis_angle(ax[0], ax[1], ax[2], q[i], rot);
            m3mul(r1, rot, c->R[i]);
            c->p[i][0] = p1x; c->p[i][1] = p1y; c->p[i][2] = p1z;
        } else {
            memcpy(c->R[i], r1, sizeof r1);
            c->p[i][0] = p1x + aw[0] * q[i];
            c->p[i][1] = p1y + aw[1] * q[i];
            c->p[i][2] = p1z + aw[2] * q[i];
        }
        memcpy(pr, c->R[i], sizeof pr);
        px = c->p[i][0]; py = c->p[i][1]; pz = c->p[i][2];
    }
}

static void ee_from_chain(const orc_robot *rb, const chain_t *c, double *out7)
{
    int e = rb->ee;
    out7[0] = c->p[e][0]; out7[1] = c->p[e][1]; out7[2] = c->p[e][2];
    quat_of(c->R[e], out7 + 3);
}

static void spheres_from_chain(const orc_robot *rb, const chain_t *c, double *out4)
{
    for (int k = 0; k < rb->ns; k++) {
        int l = rb->sphere_link[k];
        const double *lc = rb->sphere_local + 3 * k;
        double w[3];
        m3vec(c->R[l], lc[0], lc[1], lc[2], w);
        out4[4 * k + 0] = w[0] + c->p[l][0];
        out4[4 * k + 1] = w[1] + c->p[l][1];
        out4[4 * k + 2] = w[2] + c->p[l][2];
        out4[4 * k + 3] = rb->sphere_radius[k];
    }
}

void orc_frames(const orc_robot *rb, const double *q, double *frames12)
{
    chain_t c;
    fk_chain(rb, q, &c);
    for (int i = 0; i < rb->n; i++) {
        memcpy(frames12 + 12 * i, c.R[i], 9 * sizeof(double));
        memcpy(frames12 + 12 * i + 9, c.p[i], 3 * sizeof(double));
    }
}

void orc_world_spheres(const orc_robot *rb, const double *q, double *out4)
{
    chain_t c;
    fk_chain(rb, q, &c);
    spheres_from_chain(rb, &c, out4);
}

void orc_ee_pose(const orc_robot *rb, const double *q, double *out7)
{
    chain_t c;
    fk_chain(rb, q, &c);
    ee_from_chain(rb, &c, out7);
}

/* ------------------------------------------------------------------ */
/* task error / Jacobian (pure.py:312-427)                             */
/* ------------------------------------------------------------------ */

/* relative rotation q_fixed^-1 * q_ee as a scaled rotation vector;
 * returns k and writes the (sign-canonical) vector part. */
static double rel_rotvec(const orc_spec *s, const double *qee, double *v)
{
    double r[4];
    qmul(s->q_fixed[0], -s->q_fixed[1], -s->q_fixed[2], -s->q_fixed[3],
         qee[0], qee[1], qee[2], qee[3], r);
    if (r[0] < 0.0) {
        r[0] = -r[0]; r[1] = -r[1]; r[2] = -r[2]; r[3] = -r[3];
    }
    double vn = sqrt((r[1] * r[1] + r[2] * r[2]) + r[3] * r[3]);
    v[0] = r[1]; v[1] = r[2]; v[2] = r[3];
    if (vn < 1e-12) return 2.0;
    return 2.0 * atan2(vn, r[0]) / vn;
}

static int err_from_pose(const orc_spec *s, const double *pose, double *e)
{
    int m = 0;
    double px = pose[0], py = pose[1], pz = pose[2];
    if (s->kind == 0) {
        e[m++] = ((s->anchor[0] * px + s->anchor[1] * py) + s->anchor[2] * pz) - s->offset;
    } else {
        double dx = px - s->anchor[0], dy = py - s->anchor[1], dz = pz - s->anchor[2];
        e[m++] = (s->b1[0] * dx + s->b1[1] * dy) + s->b1[2] * dz;
        e[m++] = (s->b2[0] * dx + s->b2[1] * dy) + s->b2[2] * dz;
    }
    if (s->has_orient) {
        double v[3];
        double k = rel_rotvec(s, pose + 3, v);
        e[m++] = s->weight * (k * v[0]);
        e[m++] = s->weight * (k * v[1]);
        e[m++] = s->weight * (k * v[2]);
    }
    return m;
}

int orc_task_error_at(const orc_spec *s, const double *pose7, double *e)
{
    return err_from_pose(s, pose7, e);
}

/* inverse left Jacobian of SO(3) (pure.py:348-366) */
static void so3_rate(double p0, double p1, double p2, double *a)
{
    double c2;
    double t2 = (p0 * p0 + p1 * p1) + p2 * p2;
    if (t2 < 1e-8) {
        c2 = 1.0 / 12.0 + t2 / 720.0;
    } else {
        double th = sqrt(t2);
        c2 = 1.0 / t2 - (1.0 + cos(th)) / ((2.0 * th) * sin(th));
    }
    double h0 = 0.5 * p0, h1 = 0.5 * p1, h2 = 0.5 * p2;
    double c01 = c2 * (p0 * p1), c02 = c2 * (p0 * p2), c12 = c2 * (p1 * p2);
    a[0] = 1.0 - c2 * (p1 * p1 + p2 * p2); a[1] = h2 + c01; a[2] = c02 - h1;
    a[3] = c01 - h2; a[4] = 1.0 - c2 * (p0 * p0 + p2 * p2); a[5] = h0 + c12;
    a[6] = h1 + c02; a[7] = c12 - h0; a[8] = 1.0 - c2 * (p0 * p0 + p1 * p1);
}

static int err_jac_from_chain(const orc_spec *s, const orc_robot *rb,
                              const chain_t *c, double *e, double *J)
{
    double pose[7];
    ee_from_chain(rb, c, pose);
    int m = err_from_pose(s, pose, e);
    int n = rb->n;
    double lin[MAXN][3], ang[MAXN][3];
    for (int j = 0; j < n; j++) {
        const double *a = c->axis_w[j];
        if (rb->jtypes[j] == 0) {
            double rx = pose[0] - c->org_w[j][0];
            double ry = pose[1] - c->org_w[j][1];
            double rz = pose[2] - c->org_w[j][2];
            lin[j][0] = a[1] * rz - a[2] * ry;
            lin[j][1] = a[2] * rx - a[0] * rz;
            lin[j][2] = a[0] * ry - a[1] * rx;
            ang[j][0] = a[0]; ang[j][1] = a[1]; ang[j][2] = a[2];
        } else {
            lin[j][0] = a[0]; lin[j][1] = a[1]; lin[j][2] = a[2];
            ang[j][0] = 0.0; ang[j][1] = 0.0; ang[j][2] = 0.0;
        }
    }
    int row = 0;
    if (s->kind == 0) {
        for (int j = 0; j < n; j++)
            J[row * n + j] = (s->anchor[0] * lin[j][0] + s->anchor[1] * lin[j][1]) +
                             s->anchor[2] * lin[j][2];
        row++;
    } else {
        for (int j = 0; j < n; j++)
            J[row * n + j] = (s->b1[0] * lin[j][0] + s->b1[1] * lin[j][1]) + s->b1[2] * lin[j][2];
        row++;
        for (int j = 0; j < n; j++)
            J[row * n + j] = (s->b2[0] * lin[j][0] + s->b2[1] * lin[j][1]) + s->b2[2] * lin[j][2];
        row++;
    }
    if (s->has_orient) {
        double v[3], a[9], mm[9];
        double k = rel_rotvec(s, pose + 3, v);
        so3_rate(k * v[0], k * v[1], k * v[2], a);
        m3mul(a, s->r_fixed_t, mm);
        for (int r = 0; r < 3; r++) {
            double m0 = s->weight * mm[3 * r];
            double m1 = s->weight * mm[3 * r + 1];
            double m2 = s->weight * mm[3 * r + 2];
            for (int j = 0; j < n; j++)
                J[row * n + j] = (m0 * ang[j][0] + m1 * ang[j][1]) + m2 * ang[j][2];
            row++;
        }
    }
    return m;
}

int orc_task_err_jac(const orc_spec *s, const orc_robot *rb, const double *q,
                     double *e, double *J)
{
    chain_t c;
    fk_chain(rb, q, &c);
    return err_jac_from_chain(s, rb, &c, e, J);
}

/* J^T (J J^T + lam^2 I)^-1 e by Cholesky; 0 if not SPD (pure.py:437-480) */
int orc_damped_step(int m, int n, const double *J, const double *e, double lam,
                    double *step)
{
    double A[MAXM][MAXM], L[MAXM][MAXM], y[MAXM], z[MAXM];
    for (int i = 0; i < m; i++) {
        for (int j = 0; j <= i; j++) {
            double acc = 0.0;
            for (int k = 0; k < n; k++) acc += J[i * n + k] * J[j * n + k];
            A[i][j] = acc;
        }
        A[i][i] += lam * lam;
    }
    for (int i = 0; i < m; i++) {
        for (int j = 0; j <= i; j++) {
            double acc = A[i][j];
            for (int k = 0; k < j; k++) acc -= L[i][k] * L[j][k];
            if (i == j) {
                if (acc <= 0.0) return 0;
                L[i][i] = sqrt(acc);
            } else {
                L[i][j] = acc / L[j][j];
            }
        }
    }
    for (int i = 0; i < m; i++) {
        double acc = e[i];
        for (int k = 0; k < i; k++) acc -= L[i][k] * y[k];
        y[i] = acc / L[i][i];
    }
    for (int i = m - 1; i >= 0; i--) {
        double acc = y[i];
        for (int k = i + 1; k < m; k++) acc -= L[k][i] * z[k];
        z[i] = acc / L[i][i];
    }
    for (int k = 0; k < n; k++) step[k] = 0.0;
    for (int i = 0; i < m; i++)
        for (int k = 0; k < n; k++) step[k] += J[i * n + k] * z[i];
    return 1;
}

/* ------------------------------------------------------------------ */
/* segment projection (pure.py:511-635)                                */
/* ------------------------------------------------------------------ */

static double err_norm_seq(const double *e, int m)
{
    double acc = 0.0;
    for (int i = 0; i < m; i++) acc += e[i] * e[i];
    return sqrt(acc);
}

/* one worker's stage-1 update (pure.py:511-546) */
static int stage1(const orc_robot *rb, const orc_spec *s, const double *xt,
                  const double *xp, double tau_task, double tau_sm,
                  double alpha, double lam, double *xnew)
{
    int n = rb->n;
    for (int k = 0; k < n; k++) {
        if (!isfinite(xt[k])) {
            memcpy(xnew, xt, n * sizeof(double));
            return 0;
        }
    }
    chain_t c;
    double e[MAXM], J[MAXM * MAXN], g[MAXN], diff[MAXN];
    fk_chain(rb, xt, &c);
    int m = err_jac_from_chain(s, rb, &c, e, J);
    double en = err_norm_seq(e, m);
    if (!orc_damped_step(m, n, J, e, lam, g))
        for (int k = 0; k < n; k++) g[k] = 0.0;
    double acc = 0.0;
    for (int k = 0; k < n; k++) {
        double d = xt[k] - xp[k];
        diff[k] = d;
        acc += d * d;
    }
    double gap = sqrt(acc);
    double exc = gap - tau_sm;
    if (exc < 0.0) exc = 0.0;
    for (int k = 0; k < n; k++) xnew[k] = xt[k] - alpha * (g[k] + diff[k] * exc);
    return gap < tau_sm && en < tau_task;
}

int orc_project_segment(const orc_robot *rb, const orc_spec *s, int w,
                        const double *wps, double tau_task, double tau_sm,
                        double alpha, double lam, int max_iters, int mode,
                        double *xi, int *iters, int *prog_out,
                        double *trace_xi, int *trace_prog, int *trace_len)
{
    int n = rb->n;
    memcpy(xi, wps, (size_t)w * n * sizeof(double));
    if (trace_len) *trace_len = 0;
    if (mode == 2) {
        /* sequential baseline (pure.py:580-615) */
        int total = 0;
        double q[MAXN], e[MAXM], J[MAXM * MAXN], st[MAXN];
        for (int t = 1; t < w; t++) {
            memcpy(q, xi + t * n, n * sizeof(double));
            int it = 0;
            for (;;) {
                for (int k = 0; k < n; k++)
                    if (!isfinite(q[k])) goto fail_seq;
                int m = orc_task_err_jac(s, rb, q, e, J);
                if (err_norm_seq(e, m) < tau_task) break;
                if (it == max_iters) goto fail_seq;
                if (!orc_damped_step(m, n, J, e, lam, st)) goto fail_seq;
                for (int k = 0; k < n; k++) q[k] = q[k] - alpha * st[k];
                it++;
            }
            total += it;
            {
                double acc = 0.0;
                for (int k = 0; k < n; k++) {
                    double d = q[k] - xi[(t - 1) * n + k];
                    acc += d * d;
                }
                if (sqrt(acc) >= tau_sm) goto fail_seq;
            }
            memcpy(xi + t * n, q, n * sizeof(double));
            continue;
fail_seq:
            *iters = max_iters;
            *prog_out = t - 1;
            return 0;
        }
        *iters = total;
        *prog_out = w - 1;
        return 1;
    }
    /* parallel / literal-gap (pure.py:549-577) */
    double *xnew = malloc((size_t)w * n * sizeof(double));
    int *valid = calloc((size_t)w, sizeof(int));
    memcpy(xnew, xi, (size_t)w * n * sizeof(double));
    int prog = 0;
    for (int it = 1; it <= max_iters; it++) {
        for (int t = prog + 1; t < w; t++)
            valid[t] = stage1(rb, s, xi + t * n, xi + (t - 1) * n, tau_task,
                              tau_sm, alpha, lam, xnew + t * n);
        if (mode == 1) {
            for (int j = prog + 1; j < w; j++)
                if (valid[j]) prog = j;
        } else {
            int j = prog + 1;
            while (j < w && valid[j]) {
                prog = j;
                j++;
            }
        }
        if (prog == w - 1) {
            if (trace_xi) {
                memcpy(trace_xi + (size_t)(*trace_len) * w * n, xi, (size_t)w * n * sizeof(double));
                trace_prog[*trace_len] = prog;
                (*trace_len)++;
            }
            *iters = it;
            *prog_out = prog;
            free(xnew);
            free(valid);
            return 1;
        }
        for (int t = prog + 1; t < w; t++)
            memcpy(xi + t * n, xnew + t * n, n * sizeof(double));
        if (trace_xi) {
            memcpy(trace_xi + (size_t)(*trace_len) * w * n, xi, (size_t)w * n * sizeof(double));
            trace_prog[*trace_len] = prog;
            (*trace_len)++;
        }
    }
    *iters = max_iters;
    *prog_out = prog;
    free(xnew);
    free(valid);
    return 0;
}

/* ------------------------------------------------------------------ */
/* motion validation, lockstep round robin (pure.py:646-699)           */
/* ------------------------------------------------------------------ */

static double check_clearance(const orc_robot *rb, const orc_scene *sc,
                              const double *sp, int64_t rnd, int env)
{
    if (rnd < (int64_t)rb->ns * env) {
        int si = (int)(rnd / env);
        int pi = (int)(rnd - (int64_t)si * env);
        const double *c = sp + 4 * si;
        if (pi < sc->nb) {
            const double *lo = sc->box_min + 3 * pi, *hi = sc->box_max + 3 * pi;
            return orc_sphere_aabb_clearance(c[0], c[1], c[2], c[3], lo[0], lo[1],
                                             lo[2], hi[0], hi[1], hi[2]);
        }
        const double *oc = sc->sph_center + 3 * (pi - sc->nb);
        return orc_sphere_sphere_clearance(c[0], c[1], c[2], c[3], oc[0], oc[1],
                                           oc[2], sc->sph_radius[pi - sc->nb]);
    }
    int k = (int)(rnd - (int64_t)rb->ns * env);
    const double *a = sp + 4 * rb->pairs[2 * k], *b = sp + 4 * rb->pairs[2 * k + 1];
    return orc_sphere_sphere_clearance(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3]);
}

int orc_validate_waypoints(const orc_robot *rb, const orc_scene *sc, int w,
                           const double *wps, int flag_on, int64_t *performed,
                           int64_t *possible, int *first_bad)
{
    int n = rb->n, env = sc->nb + sc->ne;
    int64_t per = (int64_t)rb->ns * env + rb->np;
    double *sp = malloc((size_t)(w > 0 ? w : 1) * (rb->ns > 0 ? rb->ns : 1) * 4 * sizeof(double));
    char *have = calloc((size_t)(w > 0 ? w : 1), 1);
    int64_t perf = 0;
    int flag = 0, fb = -1;
    for (int64_t rnd = 0; rnd < per; rnd++) {
        if (flag_on && flag) break;
        for (int t = 0; t < w; t++) {
            if (flag_on && flag) break;
            double *spt = sp + (size_t)t * rb->ns * 4;
            if (!have[t]) {
                orc_world_spheres(rb, wps + (size_t)t * n, spt);
                have[t] = 1;
            }
            double c = check_clearance(rb, sc, spt, rnd, env);
            perf++;
            if (c < 0.0) {
                if (fb < 0) fb = t;
                flag = 1;
            }
        }
    }
    free(sp);
    free(have);
    *performed = perf;
    *possible = (int64_t)w * per;
    *first_bad = fb;
    return fb < 0;
}

/* ------------------------------------------------------------------ */
/* Halton sampling (sampling.py:32-81)                                 */
/* ------------------------------------------------------------------ */

double orc_radical_inverse(int64_t index, int base)
{
    double f = 0.0;
    double scale = 1.0 / base;
    int64_t i = index;
    while (i > 0) {
        f += (double)(i % base) * scale;
        scale /= base;
        i /= base;
    }
    return f;
}

static int nth_prime(int k)
{
    int found = 0;
    for (int c = 2;; c++) {
        int ok = 1;
        for (int d = 2; d * d <= c; d++)
            if (c % d == 0) {
                ok = 0;
                break;
            }
        if (ok && found++ == k) return c;
    }
}

void orc_halton(int n, int64_t index, int64_t seed_offset, const double *lo,
                const double *hi, double *out)
{
    for (int k = 0; k < n; k++) {
        double u = orc_radical_inverse(index + seed_offset, nth_prime(k));
        out[k] = lo[k] + (hi[k] - lo[k]) * u;
    }
}

/* nearest: argmin of squared distance, lowest index on ties (planner.py:198-201) */
int orc_nearest(int count, int n, const double *nodes, const double *q)
{
    int best = 0;
    double bd = 0.0;
    for (int i = 0; i < count; i++) {
        double d = sqnorm_diff_np(nodes + (size_t)i * n, q, n);
        if (i == 0 || d < bd || (isnan(d) && !isnan(bd))) {
            bd = d;
            best = i;
        }
    }
    return best;
}

/* ------------------------------------------------------------------ */
/* planner (planner.py:42-505, projection.py:114-213)                  */
/* ------------------------------------------------------------------ */

typedef struct {
    double *buf;
    int32_t *parent;
    int len, cap, n;
} tree_t;

static void tree_init(tree_t *t, const double *root, int n)
{
    t->n = n;
    t->cap = 64;
    t->len = 1;
    t->buf = malloc((size_t)t->cap * n * sizeof(double));
    t->parent = malloc((size_t)t->cap * sizeof(int32_t));
    memcpy(t->buf, root, n * sizeof(double));
    t->parent[0] = 0;
}

static int tree_add(tree_t *t, const double *q, int parent)
{
    if (t->len == t->cap) {
        t->cap *= 2;
        t->buf = realloc(t->buf, (size_t)t->cap * t->n * sizeof(double));
        t->parent = realloc(t->parent, (size_t)t->cap * sizeof(int32_t));
    }
    memcpy(t->buf + (size_t)t->len * t->n, q, t->n * sizeof(double));
    t->parent[t->len] = parent;
    return t->len++;
}

static void tree_free(tree_t *t)
{
    free(t->buf);
    free(t->parent);
}

typedef struct {
    const orc_robot *rb;
    const orc_scene *sc;
    const orc_spec *sp;
    const orc_params *p;
    double spec_tau;
    int64_t st[7]; /* iterations, att, added, pfail, crej, ccperf, ccposs */
} ctx_t;

static int eqv(const double *a, const double *b, int n)
{
    for (int k = 0; k < n; k++)
        if (!(a[k] == b[k])) return 0;
    return 1;
}

/* steer (planner.py:204-211) */
static void steer(const double *qn, const double *qr, double step, int n, double *out)
{
    double d[MAXN], sq[MAXN];
    for (int k = 0; k < n; k++) {
        d[k] = qr[k] - qn[k];
        sq[k] = d[k] * d[k];
    }
    double dist = sqrt(orc_np_sum(sq, n));
    if (dist <= step) {
        memcpy(out, qr, n * sizeof(double));
        return;
    }
    double f = step / dist;
    for (int k = 0; k < n; k++) out[k] = qn[k] + f * d[k];
}

/* interpolate_segment (projection.py:114-128) */
static void interpolate(const double *a, const double *b, int w, int n, double *wp)
{
    double d[MAXN];
    for (int k = 0; k < n; k++) d[k] = b[k] - a[k];
    for (int t = 0; t < w; t++) {
        double f = (double)t / (double)(w - 1);
        for (int k = 0; k < n; k++) wp[t * n + k] = a[k] + f * d[k];
    }
    memcpy(wp, a, n * sizeof(double));
    memcpy(wp + (w - 1) * n, b, n * sizeof(double));
}

/* _resolve_taus (projection.py:137-144) */
static void resolve_taus(const ctx_t *c, const double *wp, int w, double *tt, double *ts)
{
    int n = c->rb->n;
    *tt = isnan(c->p->tau_task) ? c->spec_tau : c->p->tau_task;
    if (!isnan(c->p->tau_sm)) {
        *ts = c->p->tau_sm;
        return;
    }
    double gmax = -INFINITY;
    for (int t = 1; t < w; t++) {
        double g = sqrt(sqnorm_diff_np(wp + t * n, wp + (t - 1) * n, n));
        if (g > gmax || isnan(g)) gmax = g;
    }
    *ts = gmax > 0 ? 1.5 * gmax : 1e-6;
}

/* _recheck (projection.py:147-159) */
static int recheck(const ctx_t *c, const double *xi, int w, double tt, double ts)
{
    int n = c->rb->n;
    for (int t = 0; t < w; t++) {
        double pose[7], e[MAXM];
        orc_ee_pose(c->rb, xi + t * n, pose);
        int m = err_from_pose(c->sp, pose, e);
        double sq[MAXM];
        for (int i = 0; i < m; i++) sq[i] = e[i] * e[i];
        if (!(sqrt(orc_np_sum(sq, m)) < tt)) return 0;
        if (t > 0 && !(sqrt(sqnorm_diff_np(xi + t * n, xi + (t - 1) * n, n)) < ts)) return 0;
    }
    return 1;
}

/* parallel_project / sequential_project + _finish (projection.py:162-228);
 * xi (w*n) in/out. */
static int project(const ctx_t *c, double *xi, int w)
{
    int n = c->rb->n;
    double tt, ts;
    resolve_taus(c, xi, w, &tt, &ts);
    double *out = malloc((size_t)w * n * sizeof(double));
    int iters, prog;
    int ok = orc_project_segment(c->rb, c->sp, w, xi, tt, ts, c->p->alpha, c->p->lam,
                                 c->p->proj_max_iters, c->p->projection_mode, out,
                                 &iters, &prog, NULL, NULL, NULL);
    if (ok) {
        double *cl = malloc((size_t)w * n * sizeof(double));
        int changed = 0;
        for (int t = 0; t < w; t++)
            for (int k = 0; k < n; k++) {
                double v = out[t * n + k];
                double lo = c->rb->lo[k], hi = c->rb->hi[k];
                double r = v < lo ? lo : v;
                r = r > hi ? hi : r;
                cl[t * n + k] = r;
                if (!(r == v)) changed = 1;
            }
        if (changed) {
            if (recheck(c, cl, w, tt, ts))
                memcpy(out, cl, (size_t)w * n * sizeof(double));
            else
                ok = 0;
        }
        free(cl);
    }
    memcpy(xi, out, (size_t)w * n * sizeof(double));
    free(out);
    return ok;
}

static int validate(ctx_t *c, const double *wp, int w, int64_t *perf, int64_t *poss)
{
    int fb;
    return orc_validate_waypoints(c->rb, c->sc, w, wp, c->p->flag_on, perf, poss, &fb);
}

/* derive_edge (planner.py:223-245); counters into d[3..6] if d != NULL */
static int derive_edge(ctx_t *c, const double *a, const double *b, int64_t *d)
{
    int w = c->p->width, n = c->rb->n;
    double *wp = malloc((size_t)w * n * sizeof(double));
    interpolate(a, b, w, n, wp);
    int ok = project(c, wp, w);
    if (!ok) {
        if (d) d[3] += 1;
        free(wp);
        return 0;
    }
    int64_t pf, ps;
    int v = validate(c, wp, w, &pf, &ps);
    if (d) {
        d[5] += pf;
        d[6] += ps;
    }
    free(wp);
    if (!v) {
        if (d) d[4] += 1;
        return 0;
    }
    return 1;
}

typedef struct {
    int i_near;
    double q_end[MAXN];
    int64_t pf, cr, cp, cs;
    int reason; /* 0 ok, 1 projection, 2 collision, 3 degenerate */
} attempt_t;

/* _attempt_extend (planner.py:265-306) */
static void attempt_extend(ctx_t *c, const tree_t *tr, int snap, const double *qr,
                           attempt_t *at)
{
    int n = c->rb->n, w = c->p->width;
    memset(at, 0, sizeof *at);
    at->i_near = orc_nearest(snap, n, tr->buf, qr);
    const double *qn = tr->buf + (size_t)at->i_near * n;
    double qs[MAXN];
    steer(qn, qr, c->p->step_size, n, qs);
    if (eqv(qs, qn, n)) {
        memcpy(at->q_end, qn, n * sizeof(double));
        at->reason = 3;
        return;
    }
    double *wp = malloc((size_t)w * n * sizeof(double));
    interpolate(qn, qs, w, n, wp);
    if (!project(c, wp, w)) {
        memcpy(at->q_end, qs, n * sizeof(double));
        at->pf = 1;
        at->reason = 1;
        free(wp);
        return;
    }
    memcpy(at->q_end, wp + (w - 1) * n, n * sizeof(double));
    if (eqv(at->q_end, qn, n)) {
        at->reason = 3;
        free(wp);
        return;
    }
    if (eqv(at->q_end, qs, n)) {
        int64_t pf, ps;
        int v = validate(c, wp, w, &pf, &ps);
        at->cp = pf;
        at->cs = ps;
        if (!v) {
            at->cr = 1;
            at->reason = 2;
        }
        free(wp);
        return;
    }
    free(wp);
    int64_t d[7] = {0};
    if (!derive_edge(c, qn, at->q_end, d)) {
        at->reason = d[3] ? 1 : 2;
    }
    at->pf = d[3];
    at->cr = d[4];
    at->cp = d[5];
    at->cs = d[6];
}

static void merge_attempt(ctx_t *c, const attempt_t *a)
{
    c->st[1] += 1;
    c->st[3] += a->pf;
    c->st[4] += a->cr;
    c->st[5] += a->cp;
    c->st[6] += a->cs;
}

/* connect (planner.py:361-409); returns 0 trapped/advanced, 1 reached */
static int connect(ctx_t *c, tree_t *tr, const double *qt, int *meet)
{
    int n = c->rb->n, w = c->p->width;
    int icur = orc_nearest(tr->len, n, tr->buf, qt);
    double qc[MAXN];
    memcpy(qc, tr->buf + (size_t)icur * n, n * sizeof(double));
    double dist = sqrt(sqnorm_diff_np(qc, qt, n));
    double tol = isnan(c->p->connect_tolerance) ? c->p->step_size / 10.0
                                                : c->p->connect_tolerance;
    if (dist <= tol) {
        *meet = icur;
        return 1;
    }
    double *wp = malloc((size_t)w * n * sizeof(double));
    int reached = 0;
    for (int segs = 0; segs < c->p->max_connect_segments; segs++) {
        double qs[MAXN], qe[MAXN];
        steer(qc, qt, c->p->step_size, n, qs);
        interpolate(qc, qs, w, n, wp);
        if (!project(c, wp, w)) {
            c->st[3] += 1;
            break;
        }
        memcpy(qe, wp + (w - 1) * n, n * sizeof(double));
        if (eqv(qe, qs, n)) {
            int64_t pf, ps;
            int v = validate(c, wp, w, &pf, &ps);
            c->st[5] += pf;
            c->st[6] += ps;
            if (!v) {
                c->st[4] += 1;
                break;
            }
        } else if (!derive_edge(c, qc, qe, c->st)) {
            break;
        }
        double nd = sqrt(sqnorm_diff_np(qe, qt, n));
        if (!(nd < dist)) break;
        icur = tree_add(tr, qe, icur);
        memcpy(qc, qe, n * sizeof(double));
        dist = nd;
        if (dist <= tol) {
            *meet = icur;
            reached = 1;
            break;
        }
    }
    free(wp);
    return reached;
}

static double now_ms(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* _check_endpoint (planner.py:416-427): 0 ok, 1 limits, 2 manifold, 3 collision */
static int check_endpoint(ctx_t *c, const double *q)
{
    int n = c->rb->n;
    for (int k = 0; k < n; k++)
        if (q[k] < c->rb->lo[k] || q[k] > c->rb->hi[k]) return 1;
    double pose[7], e[MAXM], sq[MAXM];
    orc_ee_pose(c->rb, q, pose);
    int m = err_from_pose(c->sp, pose, e);
    for (int i = 0; i < m; i++) sq[i] = e[i] * e[i];
    double tau = isnan(c->p->tau_task) ? c->spec_tau : c->p->tau_task;
    if (!(sqrt(orc_np_sum(sq, m)) < tau)) return 2;
    int64_t pf, ps;
    int fb;
    if (!orc_validate_waypoints(c->rb, c->sc, 1, q, 0, &pf, &ps, &fb)) return 3;
    return 0;
}

static void extract_path(const tree_t *ts, const tree_t *tg, int ms, int mg, orc_result *out)
{
    int n = ts->n;
    int ca = 1, cb = 1;
    for (int i = ms; ts->parent[i] != i; i = ts->parent[i]) ca++;
    for (int i = mg; tg->parent[i] != i; i = tg->parent[i]) cb++;
    double *pa = malloc((size_t)ca * n * sizeof(double));
    double *pb = malloc((size_t)cb * n * sizeof(double));
    int k = ca - 1;
    for (int i = ms;; i = ts->parent[i]) {
        memcpy(pa + (size_t)k * n, ts->buf + (size_t)i * n, n * sizeof(double));
        k--;
        if (ts->parent[i] == i) break;
    }
    k = 0; /* pb = reversed(chain(meet_g)): meet first, root last */
    for (int i = mg;; i = tg->parent[i]) {
        memcpy(pb + (size_t)k * n, tg->buf + (size_t)i * n, n * sizeof(double));
        k++;
        if (tg->parent[i] == i) break;
    }
    int skip = eqv(pa + (size_t)(ca - 1) * n, pb, n) ? 1 : 0;
    int len = ca + cb - skip;
    out->path_len = len;
    out->path = malloc((size_t)len * n * sizeof(double));
    out->sources = malloc((size_t)(len > 1 ? len - 1 : 1) * sizeof(int32_t));
    memcpy(out->path, pa, (size_t)ca * n * sizeof(double));
    memcpy(out->path + (size_t)ca * n, pb + (size_t)skip * n, (size_t)(cb - skip) * n * sizeof(double));
    int s = 0;
    for (int i = 0; i < ca - 1; i++) out->sources[s++] = 0;
    if (cb - skip > 0) {
        out->sources[s++] = skip ? 2 : 1;
        for (int i = 0; i < cb - skip - 1; i++) out->sources[s++] = 2;
    }
    free(pa);
    free(pb);
}

/* plan (planner.py:430-485) */
int orc_plan(const orc_robot *rb, const orc_scene *sc, const orc_spec *sp,
             const orc_params *p, const double *start, const double *goal,
             orc_result *out)
{
    int n = rb->n;
    ctx_t c = {rb, sc, sp, p, sp->tau_task, {0}};
    memset(out, 0, sizeof *out);
    double t0 = now_ms();
    int ce = check_endpoint(&c, start);
    if (ce) {
        out->status = -ce;
        return out->status;
    }
    ce = check_endpoint(&c, goal);
    if (ce) {
        out->status = -3 - ce;
        return out->status;
    }
    if (eqv(start, goal, n)) {
        out->status = ORC_SOLVED;
        out->path_len = 1;
        out->path = malloc(n * sizeof(double));
        out->sources = malloc(sizeof(int32_t));
        memcpy(out->path, start, n * sizeof(double));
        out->stats[7] = out->stats[8] = 1;
        out->wall_ms = now_ms() - t0;
        return 0;
    }
    tree_t tr[2];
    tree_init(&tr[0], start, n);
    tree_init(&tr[1], goal, n);
    int64_t hidx = 1;
    int status = ORC_ITERLIMIT;
    attempt_t *atts = malloc((size_t)p->attempts * sizeof(attempt_t));
    double *samples = malloc((size_t)p->attempts * n * sizeof(double));
    for (int it = 1; it <= p->max_iterations; it++) {
        if (!p->deterministic && now_ms() - t0 > p->time_budget_ms) {
            status = ORC_TIMEDOUT;
            break;
        }
        c.st[0] = it;
        int ai = (it - 1) % 2;
        tree_t *a = &tr[ai], *b = &tr[1 - ai];
        for (int s = 0; s < p->attempts; s++)
            orc_halton(n, hidx++, p->seed_offset, rb->lo, rb->hi, samples + (size_t)s * n);
        /* _extend_batch (planner.py:328-358) */
        int snap = a->len, nres = 0, win = -1;
        for (int s = 0; s < p->attempts; s++) {
            attempt_extend(&c, a, snap, samples + (size_t)s * n, &atts[s]);
            nres++;
            if (atts[s].reason == 0 && (p->deterministic || p->attempts == 1)) break;
        }
        for (int s = 0; s < nres; s++) {
            merge_attempt(&c, &atts[s]);
            if (win < 0 && atts[s].reason == 0) win = s;
        }
        if (win < 0) continue;
        int node = tree_add(a, atts[win].q_end, atts[win].i_near);
        c.st[2] += 1;
        double qnew[MAXN];
        memcpy(qnew, a->buf + (size_t)node * n, n * sizeof(double));
        int meet;
        if (!connect(&c, b, qnew, &meet)) continue;
        double qm[MAXN];
        memcpy(qm, b->buf + (size_t)meet * n, n * sizeof(double));
        int ms, mg;
        const double *js, *jg;
        if (ai == 0) {
            ms = node; mg = meet; js = qnew; jg = qm;
        } else {
            ms = meet; mg = node; js = qm; jg = qnew;
        }
        if (eqv(js, jg, n) || derive_edge(&c, js, jg, c.st)) {
            extract_path(&tr[0], &tr[1], ms, mg, out);
            status = ORC_SOLVED;
            break;
        }
    }
    out->status = status;
    out->wall_ms = now_ms() - t0;
    for (int k = 0; k < 7; k++) out->stats[k] = c.st[k];
    out->stats[7] = tr[0].len;
    out->stats[8] = tr[1].len;
    tree_free(&tr[0]);
    tree_free(&tr[1]);
    free(atts);
    free(samples);
    return status;
}

void orc_result_free(orc_result *res)
{
    free(res->path);
    free(res->sources);
    res->path = NULL;
    res->sources = NULL;
}
