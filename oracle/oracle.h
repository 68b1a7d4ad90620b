/*
 * oracle.h -- CPU restatement of the reference (maniplan) hot path, FP64.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 planner: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2505_06791_b200) never links or calls it.
 *
 * Every function restates the reference algorithm with the same evaluation
 * order and is compiled with -ffp-contract=off -fno-builtin-sin/cos (the
 * reference's own flags, pkg/setup.py:45-53), so results are bit-identical
 * to the reference's float64 kernels on the same libm.  Pinned against the
 * golden vectors in tests/golden/ (generated from the reference by
 * tests/golden/make_golden.py).
 */
#ifndef CPRRTC_ORACLE_H
#define CPRRTC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PackedRobot (reference kinematics.py:158-224) */
typedef struct {
    int n;                       /* joints */
    const int32_t *jtypes;       /* (n) 0 revolute, 1 prismatic */
    const double *axes;          /* (n,3) */
    const double *origin_r;      /* (n,9) row-major */
    const double *origin_p;      /* (n,3) */
    const double *lo, *hi;       /* (n) */
    int ns;                      /* spheres */
    const int32_t *sphere_link;  /* (ns) */
    const double *sphere_local;  /* (ns,3) */
    const double *sphere_radius; /* (ns) */
    int np;                      /* self pairs */
    const int32_t *pairs;        /* (np,2) */
    int ee;                      /* ee link */
} orc_robot;

/* PackedScene (reference geometry.py:101-135) */
typedef struct {
    int nb;
    const double *box_min, *box_max; /* (nb,3) */
    int ne;
    const double *sph_center;        /* (ne,3) */
    const double *sph_radius;        /* (ne) */
} orc_scene;

/* PackedConstraint (reference constraints.py:123-176) */
typedef struct {
    int kind;            /* 0 plane (anchor=normal), 1 line (anchor=point) */
    double anchor[3];
    double offset;
    double b1[3], b2[3];
    int has_orient;
    double q_fixed[4];
    double r_fixed_t[9];
    double weight;
    double tau_task;
} orc_spec;

/* PlanParams + ProjectionParams (reference planner.py:88-112, projection.py:75-90) */
typedef struct {
    double step_size;
    int width;
    double alpha;
    int proj_max_iters;
    double lam;
    double tau_task;          /* NaN -> spec tau */
    double tau_sm;            /* NaN -> auto (1.5 x max initial gap) */
    int max_iterations;
    double time_budget_ms;
    double connect_tolerance; /* NaN -> step/10 */
    int projection_mode;      /* 0 parallel, 1 literal-gap, 2 naive */
    int flag_on;
    int64_t seed_offset;
    int deterministic;
    int attempts;
    int max_connect_segments;
} orc_params;

enum { ORC_SOLVED = 0, ORC_TIMEDOUT = 1, ORC_ITERLIMIT = 2 };

typedef struct {
    int status;               /* ORC_* or negative setup error (-1..-6) */
    int path_len;
    double *path;             /* (path_len, n), malloc'd */
    int32_t *sources;         /* (path_len-1): 0 start, 1 junction, 2 goal */
    int64_t stats[9];         /* iterations, ext_attempted, ext_added, proj_fail,
                                 coll_rej, cc_performed, cc_possible,
                                 nodes_start, nodes_goal */
    double wall_ms;
} orc_result;

double orc_sphere_aabb_clearance(double cx, double cy, double cz, double r,
                                 double lx, double ly, double lz,
                                 double hx, double hy, double hz);
double orc_sphere_sphere_clearance(double ax, double ay, double az, double ar,
                                   double bx, double by, double bz, double br);
void orc_rot_from_quat(double w, double x, double y, double z, double *out);
void orc_frames(const orc_robot *r, const double *q, double *frames12);
void orc_world_spheres(const orc_robot *r, const double *q, double *out4);
void orc_ee_pose(const orc_robot *r, const double *q, double *out7);
int orc_task_error_at(const orc_spec *s, const double *pose7, double *e);
int orc_task_err_jac(const orc_spec *s, const orc_robot *r, const double *q,
                     double *e, double *jac /* m x n row-major */);
int orc_damped_step(int m, int n, const double *jac, const double *e,
                    double lam, double *step);
int orc_project_segment(const orc_robot *r, const orc_spec *s, int w,
                        const double *wps, double tau_task, double tau_sm,
                        double alpha, double lam, int max_iters, int mode,
                        double *xi_out, int *iters, int *prog,
                        double *trace_xi, int *trace_prog, int *trace_len);
int orc_validate_waypoints(const orc_robot *r, const orc_scene *sc, int w,
                           const double *wps, int flag_on, int64_t *performed,
                           int64_t *possible, int *first_bad);
double orc_radical_inverse(int64_t index, int base);
void orc_halton(int n, int64_t index, int64_t seed_offset, const double *lo,
                const double *hi, double *out);
int orc_nearest(int count, int n, const double *nodes, const double *q);
double orc_np_sum(const double *a, int n);
int orc_plan(const orc_robot *r, const orc_scene *sc, const orc_spec *s,
             const orc_params *p, const double *start, const double *goal,
             orc_result *out);
void orc_result_free(orc_result *res);

#ifdef __cplusplus
}
#endif
#endif
