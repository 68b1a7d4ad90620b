/*
 * cprrtc.h -- C ABI of the B200-native cpRRTC planner (libcprrtc.so).
 *
 * Plain pointers and sizes only; FP64 host buffers in and out (the device
 * computes in FP32 on the planning hot path, FP64 for setup checks).  The
 * caller owns every host buffer; a context owns its device memory, CUDA
 * stream and NVRTC-compiled modules.  Calls are synchronous on the context's
 * stream.  One context per (host thread, GPU).  Every function returns 0 on
 * success and a negative CPRRTC_E* code on failure; cprrtc_last_error()
 * gives the message (thread-local).
 *
 * Each entry point replaces one function of the reference's kernel-backend
 * protocol (maniplan/_kernels, selected at maniplan/_kernels/__init__.py:33-44)
 * or of its planner (maniplan/planner.py); the citation is next to it.  The
 * reference binds those through Python; INTEGRATION.md shows the ctypes stub
 * a maintainer adds to select this library as a backend.
 */
#ifndef CPRRTC_H
#define CPRRTC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPRRTC_ABI_VERSION 2

#if defined(__GNUC__)
#define CPRRTC_API __attribute__((visibility("default")))
#else
#define CPRRTC_API
#endif

enum {
    CPRRTC_OK = 0,
    CPRRTC_EARG = -1,      /* bad argument (maps to ValueError) */
    CPRRTC_ECUDA = -2,     /* CUDA runtime / driver failure */
    CPRRTC_ENVRTC = -3,    /* NVRTC compile failure */
    CPRRTC_ENODEV = -4,    /* no CUDA device */
    CPRRTC_ESINGULAR = -5, /* undamped solve hit a singular J J^T */
    CPRRTC_ELIMIT = -6     /* a size exceeds a compiled capacity */
};

/* PackedRobot (maniplan/kinematics.py:158-224) */
typedef struct {
    int n;
    const int32_t *jtypes;       /* (n) 0 revolute, 1 prismatic */
    const double *axes;          /* (n,3) */
    const double *origin_r;      /* (n,9) row-major */
    const double *origin_p;      /* (n,3) */
    const double *lo, *hi;       /* (n) */
    int n_spheres;
    const int32_t *sphere_link;  /* (S) */
    const double *sphere_local;  /* (S,3) */
    const double *sphere_radius; /* (S) */
    int n_pairs;
    const int32_t *pairs;        /* (P,2) */
    int ee_link;
} cprrtc_robot;

/* PackedScene (maniplan/geometry.py:101-135) */
typedef struct {
    int n_boxes;
    const double *box_min, *box_max; /* (B,3) */
    int n_spheres;
    const double *sph_center;        /* (E,3) */
    const double *sph_radius;        /* (E) */
} cprrtc_scene;

/* PackedConstraint (maniplan/constraints.py:123-176) */
typedef struct {
    int kind;             /* 0 plane, 1 line */
    double anchor[3];     /* plane normal / line point */
    double offset;
    double basis[6];      /* (2,3) line basis */
    int has_orient;
    double q_fixed[4];
    double r_fixed_t[9];
    double weight;
    double tau_task;      /* +inf: unconstrained (constraints.py:179-186) */
} cprrtc_constraint;

/* PlanParams + ProjectionParams (maniplan/planner.py:88-112,
 * maniplan/projection.py:75-90) plus device knobs. */
typedef struct {
    double step_size;
    int width;               /* waypoints per motion, 2..32 */
    double alpha;
    int proj_max_iters;
    double lam;
    double tau_task;         /* <= 0: from the constraint */
    double tau_sm;           /* <= 0: auto, 1.5 x max initial gap */
    int max_iterations;      /* samples drawn, across all teams */
    double time_budget_ms;   /* deterministic: ignored; <= 0: expired (TimedOut before sample 1, planner.py:450-453) */
    double connect_tolerance;/* <= 0: step_size / 10 */
    int projection_mode;     /* 0 parallel, 1 literal-gap, 2 naive */
    int flag_on;
    int deterministic;
    int max_connect_segments;
    double cc_margin;        /* robot-sphere inflation in the planner (m) */
    int teams;               /* concurrent extension teams (0: fill the GPU) */
    int tree_capacity;       /* nodes per tree (0: auto) */
    int path_capacity;       /* max path nodes returned per query (0: 1024) */
    int cc_broadphase;       /* 1: planner CC through the clustered broad phase
                                (cprrtc_validate_broadphase; same verdicts, the
                                cc_performed stat then counts evaluated checks);
                                0: the reference's lockstep check order;
                                -1: on whenever the scene has obstacles */
} cprrtc_params;

/* stats[] layout of cprrtc_result (PlanStats, planner.py:130-141) */
enum {
    CPRRTC_ST_ITERATIONS = 0, CPRRTC_ST_EXT_ATTEMPTED, CPRRTC_ST_EXT_ADDED,
    CPRRTC_ST_PROJ_FAIL, CPRRTC_ST_COLL_REJECT, CPRRTC_ST_CC_PERFORMED,
    CPRRTC_ST_CC_POSSIBLE, CPRRTC_ST_GPU_CHECKS,
    /* device work units (roofline accounting) */
    CPRRTC_ST_STAGE1_EVALS, CPRRTC_ST_CC_FK_EVALS, CPRRTC_ST_NN_NODES, CPRRTC_ST_PROJ_ITERS,
    CPRRTC_ST_COUNT
};

typedef struct {
    int status;          /* 0 Solved, 1 TimedOut, 2 IterLimit, 3 tree full,
                            4 path longer than path_capacity, 5 stopped because
                            another racer solved (cprrtc_plan_race), -1 setup error */
    int setup_code;      /* 0 ok; 1/2/3 start limits/manifold/collision;
                            4/5/6 the same for the goal (planner.py:416-427) */
    int path_len;
    int nodes_start, nodes_goal;
    double device_ms;    /* device time of this query (globaltimer) */
    uint64_t stats[CPRRTC_ST_COUNT];
} cprrtc_result;

CPRRTC_API int cprrtc_abi_version(void);
CPRRTC_API const char *cprrtc_last_error(void);
CPRRTC_API int cprrtc_device_count(int *count);

/* Emit the robot-specialised CUDA source (unrolled FK, constants) that
 * NVRTC compiles; usable without a GPU.  *needed = bytes incl. NUL. */
CPRRTC_API int cprrtc_codegen(const cprrtc_robot *robot, char *buf, size_t cap, size_t *needed);

/* NVRTC-compile the planner (parity=0) or parity/batch-kernel (parity=1)
 * module for (team width G in {16,32}, constraint kind, orientation lock) into the on-disk cubin cache without a GPU
 * (build-time warm-up); path receives the cubin file name. */
CPRRTC_API int cprrtc_precompile(const cprrtc_robot *robot, int G, int kind, int orient, int parity,
                                 char *path, size_t cap);
/* the full NVRTC translation unit for that module (for offline nvcc checks) */
CPRRTC_API int cprrtc_device_source(const cprrtc_robot *robot, int G, int kind, int orient, int parity,
                                    char *buf, size_t cap, size_t *needed);

CPRRTC_API int cprrtc_ctx_create(int device, const cprrtc_robot *robot, void **ctx);
CPRRTC_API int cprrtc_ctx_destroy(void *ctx);
/* scene / constraint of subsequent calls; constraint NULL = unconstrained */
CPRRTC_API int cprrtc_set_scene(void *ctx, const cprrtc_scene *scene);
CPRRTC_API int cprrtc_set_constraint(void *ctx, const cprrtc_constraint *con);
/* compile + load the module for the current constraint kind and width now
 * (NVRTC time stays out of timed regions; cached on disk) */
CPRRTC_API int cprrtc_prepare(void *ctx, int width);
/* launches of this library's kernels since context creation */
CPRRTC_API int64_t cprrtc_launch_count(void *ctx);
/* device time of the last cprrtc_plan: whole call / plan kernel.  Batches:
 * CUDA events (H2D copy -> results; the planner kernel).  A single query (its
 * lean graph records no events): the planner's own clock, init -> the result
 * complete / init -> solved.  cprrtc_plan returns for a single query as soon
 * as its result is complete (completion words in mapped memory), before the
 * planner grid retires; later calls on the context are stream-ordered.  A
 * launch that completes without writing its completion words is an error
 * (CPRRTC_ECUDA), never a stale result. */
CPRRTC_API int cprrtc_last_timing(void *ctx, double *total_ms, double *plan_kernel_ms);
/* overwrite `bytes` of device scratch (L2 flush between timed iterations) */
CPRRTC_API int cprrtc_flush_l2(void *ctx, size_t bytes);

/* frames / world spheres / ee_pose  (maniplan/_kernels/pure.py:251-271) */
CPRRTC_API int cprrtc_fk(void *ctx, int B, const double *q, int fp64, double *frames,
              double *axes, double *origins, double *ee, double *spheres);
/* task_err_jac (pure.py:490-493); e (B,M), J (B,M,n) */
CPRRTC_API int cprrtc_task_err_jac(void *ctx, int B, const double *q, int fp64, double *e, double *J);
/* task_error_at (pure.py:485-487), FP64 */
CPRRTC_API int cprrtc_task_error_at(void *ctx, int B, const double *pose7, double *e);
/* project_configuration (maniplan/projection.py:231-254), FP64 Newton */
CPRRTC_API int cprrtc_project_config(void *ctx, int B, double *q_io, double tau, double lam,
                          int max_iters, int32_t *ok);
/* endpoint test of planner.py:416-427 / validate_configuration
 * (maniplan/validation.py:73-78), FP64: 0 ok, 1 limits, 2 manifold, 3 collision */
CPRRTC_API int cprrtc_check_config(void *ctx, int B, const double *q, double tau, int32_t *code);
/* validate_waypoints (pure.py:646-699): B motions of W waypoints; exact
 * reference counters (performed = lockstep-equivalent count) */
CPRRTC_API int cprrtc_validate(void *ctx, int B, int W, const double *wps, int flag_on, double margin,
                    int32_t *valid, int32_t *first_bad, int64_t *performed,
                    int64_t *possible, int64_t *gpu_checks);
/* the same verdicts (validate_waypoints, pure.py:646-699) through the
 * clustered broad phase: Morton-sorted chunks of 8 primitives behind
 * conservative bounding boxes, per-waypoint robot bounding box.  Counters
 * are this kernel's own: performed = sphere-primitive checks evaluated,
 * gpu_checks = those + bound tests, first_bad = lowest colliding waypoint. */
CPRRTC_API int cprrtc_validate_broadphase(void *ctx, int B, int W, const double *wps, int flag_on,
                    double margin, int32_t *valid, int32_t *first_bad, int64_t *performed,
                    int64_t *possible, int64_t *gpu_checks);
/* project_segment (pure.py:618-635) for B segments; tau_sm per segment
 * (NULL: auto); trace (B,max_iters,W,n) + trace_prog (B,max_iters) optional */
CPRRTC_API int cprrtc_project(void *ctx, int B, int W, const double *wps, const double *tau_sm,
                   double tau_task, double alpha, double lam, int max_iters, int mode,
                   double *xi, int32_t *ok, int32_t *iters, int32_t *prog,
                   double *trace, int32_t *trace_prog);
/* nearest (planner.py:198-201) for Q queries over N nodes (row-major) */
CPRRTC_API int cprrtc_nearest(void *ctx, int N, const double *nodes, int Q, const double *queries,
                   int32_t *idx);
/* the same scan over n_trees trees of N nodes each, query i on tree i % n_trees
 * (nodes (n_trees, N, n)); the HBM-streaming NN benchmark of bench.py.  The
 * kernel time of this and of cprrtc_validate is cprrtc_last_timing's
 * plan_kernel_ms. */
CPRRTC_API int cprrtc_nearest_trees(void *ctx, int N, int n_trees, const float *reserved,
                                    const double *nodes, int Q, const double *queries, int32_t *idx);
/* HaltonState.next_sample (maniplan/sampling.py:65-81), FP64 bit-exact:
 * rows first_index .. first_index+count-1, mapped into [lo, hi] (NULL: the
 * robot's joint limits) */
CPRRTC_API int cprrtc_halton(void *ctx, int count, int64_t first_index, int64_t seed_offset,
                             const double *lo, const double *hi, double *out);
/* plan (planner.py:430-505) for B independent queries sharing robot, scene,
 * constraint and params.  paths (B, path_capacity, n), sources
 * (B, path_capacity): 0 start, 1 junction, 2 goal.  A solved path's first
 * and last rows are the exact FP64 start and goal (the tree roots,
 * planner.py:488-505); the rows between are the FP32 tree nodes. */
CPRRTC_API int cprrtc_plan(void *ctx, const cprrtc_params *params, int B, const double *starts,
                const double *goals, const int64_t *seeds, cprrtc_result *results,
                double *paths, int32_t *sources);
/* cprrtc_plan with the solution paths packed back to back (the batched
 * queries of BASELINE configs[4]; same planner, same results):
 * offsets (B+1): query i's path nodes are paths[offsets[i] .. offsets[i+1])
 * (n doubles each) and its edge sources sources[offsets[i] ..
 * offsets[i+1]-1); flat_capacity = rows available in paths / sources
 * (CPRRTC_ELIMIT if the batch's paths need more; results are valid then). */
CPRRTC_API int cprrtc_plan_flat(void *ctx, const cprrtc_params *params, int B, const double *starts,
                                const double *goals, const int64_t *seeds, cprrtc_result *results,
                                int64_t *offsets, double *paths, int32_t *sources, int64_t flat_capacity);
/* cprrtc_plan_flat in two halves: submit launches the batch and returns at
 * once (the inputs are staged before it returns); wait collects it into the
 * packed layout of cprrtc_plan_flat.  One batch in flight per context;
 * alternating two contexts on a device overlaps a batch's slowest queries
 * with the next batch (BASELINE configs[4] as a stream of batches). */
CPRRTC_API int cprrtc_plan_submit(void *ctx, const cprrtc_params *params, int B, const double *starts,
                                  const double *goals, const int64_t *seeds);
CPRRTC_API int cprrtc_plan_wait(void *ctx, int B, cprrtc_result *results, int64_t *offsets, double *paths,
                                int32_t *sources, int64_t flat_capacity);
/* device time (CUDA events) from the start of ctx_from's last submitted batch
 * to the end of ctx_to's (same device): a pipelined stream of batches */
CPRRTC_API int cprrtc_elapsed_ms(void *ctx_from, void *ctx_to, double *ms);   /* (batches and races:
                                      a single-query launch records no events -> CPRRTC_EARG) */
/* cprrtc_plan's batch sharded over n_ctx contexts (typically one per GPU):
 * context k plans the contiguous slice [k*B/n_ctx, (k+1)*B/n_ctx); every shard
 * is launched before any is awaited, and the results land in the caller's
 * arrays exactly as cprrtc_plan would lay them out.  Independent queries, no
 * collective (BASELINE configs[4]). */
CPRRTC_API int cprrtc_plan_multi(void *const *ctxs, int n_ctx, const cprrtc_params *params, int B,
                                 const double *starts, const double *goals, const int64_t *seeds,
                                 cprrtc_result *results, double *paths, int32_t *sources);
/* One query raced on n_ctx contexts/* One query raced on n_ctx contexts (typically one per GPU; at most
 * CPRRTC_MAX_RACE): each grows its own tree pair from seeds[k] (distinct
 * Halton offsets) with the planner of cprrtc_plan; the first racer to solve
 * stores a first-solution flag into every racer's flag word (peer stores over
 * NVLink / NVSwitch when the devices have peer access, else one mapped host
 * word) and the others stop.  results / paths / sources hold n_ctx entries
 * laid out as cprrtc_plan's with B = n_ctx; *winner = the solved racer with
 * the shortest device time, or -1.  (The reference has no counterpart: it is
 * a single-core planner, maniplan/planner.py:430-485.) */
#define CPRRTC_MAX_RACE 8
CPRRTC_API int cprrtc_plan_race(void *const *ctxs, int n_ctx, const cprrtc_params *params,
                                const double *start, const double *goal, const int64_t *seeds,
                                cprrtc_result *results, double *paths, int32_t *sources,
                                int32_t *winner);
/* One reference extend() (op 0, planner.py:317-325 / _attempt_extend :265-306)
 * or connect() (op 1, planner.py:361-409) step on a caller tree: nodes (N, n),
 * parents (N); q (n) is the sample / target.  result[0]: extend -> index of
 * the new node, or -1 degenerate, -2 projection, -3 collision, -4 full;
 * connect -> meet node index (Reached) or -1.  result[1]: segments added by
 * connect; result[2]: node count afterwards.  Appended nodes / parents are
 * returned in new_nodes (max_new, n) / new_parents; stats as cprrtc_result. */
CPRRTC_API int cprrtc_step(void *ctx, const cprrtc_params *params, int op, int N, const double *nodes,
                           const int32_t *parents, const double *q, int32_t *result,
                           double *new_nodes, int32_t *new_parents, int max_new, uint64_t *stats);

/* derive_edge (planner.py:223-245) for every consecutive pair of a path:
 * nodes (n_nodes, n), sources (n_nodes-1): 0 start, 1 junction, 2 goal --
 * goal edges are derived in tree-growth direction and returned reversed
 * (revalidate_path, planner.py:508-523).  Re-deriving a path returned by
 * cprrtc_plan reproduces the planner's certified motions exactly.
 * dense (n_nodes-1, W, n), ok (n_nodes-1). */
CPRRTC_API int cprrtc_derive_edges(void *ctx, const cprrtc_params *params, int n_nodes,
                                   const double *nodes, const int32_t *sources, double *dense,
                                   int32_t *ok);

/* robot-independent helpers (device FP64) */
CPRRTC_API int cprrtc_clearance(int device, int B, int kind, const double *a, const double *b, double *out);
CPRRTC_API int cprrtc_damped_step(int device, int B, int m, int n, const double *J, const double *e,
                       double lam, double *step, int32_t *ok);

#ifdef __cplusplus
}
#endif
#endif
