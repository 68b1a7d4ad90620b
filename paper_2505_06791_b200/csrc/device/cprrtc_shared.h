// cprrtc_shared.h -- structs shared bit-for-bit by the host runtime
// (runtime.cpp) and the NVRTC device code (prepended to cprrtc_device.cuh).
// Plain C++ only: compiled by both g++/nvcc (host) and NVRTC (device).
#ifndef CPRRTC_SHARED_H
#define CPRRTC_SHARED_H

typedef unsigned long long u64;
typedef long long i64;

// packed constraint (maniplan/constraints.py:123-176)
template <class T> struct Con {
    T anchor[3];
    T offset;
    T b1[3], b2[3];
    T qf[4];
    T rft[9];
    T weight;
};

// projection parameters (maniplan/projection.py:75-90), FP32 + device margins
struct ProjArgs {
    float alpha, lam;
    float tau_task;       // reference tolerance (inf = unconstrained)
    float tau_task_dev;   // tau_task * (1 - 1e-3) - 2e-6: FP32 safety margin
    float tau_sm_fixed;   // > 0: fixed tau_sm, else auto (1.5 x max initial gap)
    int max_iters;
    int mode;             // 0 parallel, 1 literal-gap, 2 sequential ("naive")
};

// scene: boxes as centre / half extent, spheres as centre + radius (FP32).
// Two device layouts of the same primitives:
//  * reference order (box_c / box_h / sph): the lockstep check order of
//    pure.py:674-693, exact reference counters;
//  * clustered (cl, cull = 1): primitives Morton-sorted into chunks of 8, each
//    chunk led by a conservative bounding box -- box chunk k is float4
//    [bound c, bound h, 8 box c, 8 box h] at cl + 18k, sphere chunk k is
//    [bound c, bound h, 8 spheres] at cl + 18 nbc + 10k (broad phase).
struct SceneSm {
    const float4* box_c;
    const float4* box_h;
    const float4* sph;
    int nb, ne;
    const float4* cl;
    int nbc, nec;      // box / sphere chunks of the clustered layout
    int cull;          // 1: stage and check the clustered layout
    int pad_;
};

// stats / work-unit counters (the last four feed the roofline in bench.py)
enum { ST_ITER = 0, ST_ATT, ST_ADDED, ST_PFAIL, ST_CREJ, ST_CCPERF, ST_CCPOSS, ST_GPUCHK,
       ST_STAGE1, ST_FKCC, ST_NNODES, ST_PROJITER, ST_NSTAT };

// per-query planner state in HBM, one 128-byte L2 line per access pattern:
// the flags every team polls, the counters every team hits with atomics, and
// the stats added once per team -- so polling never queues behind atomics
struct alignas(128) QueryState {
    // line 0: polled flags and read-mostly state
    int solved, stop, timed_out, overflow, exhausted;
    int race_stopped;      // stopped because another racer solved the query
    int setup_code;        // endpoint check (planner.py:416-427)
    int meet[2];           // meet node in the start / goal tree
    int hwm[2];            // nodes used by the previous run (NaN refill)
    int pad0_;
    i64 seed_offset;
    u64 t0_ns, t_end_ns;
    int pad1_[14];
    // line 1: atomics
    int count[2];          // tree node counters (atomic append)
    int next_sample;       // Halton index counter (= reference iteration)
    int active;            // teams inside the query (the last one out extracts)
    int chk_code[2];       // in-kernel endpoint checks (single query): start / goal verdicts
    int chk_cnt;           // endpoint checks done
    int pad2_[25];
    // line 2: stats (one atomicAdd per team and counter)
    u64 stats[ST_NSTAT];
    u64 pad3_[16 - ST_NSTAT];
};

struct SetupArgs {
    QueryState* qs;
    const double* starts;   // (nq, CP_N)
    const double* goals;
    const i64* seeds;
    float* trees;
    int* parents;
    int cap;
    Con<double> con;
    double tau_task;
    const double* box_min;  // (nb,3) FP64 scene for the exact endpoint test
    const double* box_max;
    const double* sph_c;
    const double* sph_r;
    int nb, ne;
    int* counters;          // planner queue counters, zeroed by block 0 (may be null)
    struct QueryOut* out;   // endpoint-check codes go straight to the results
};

struct PlanArgs {
    QueryState* qs;
    float* trees;          // (nq, 2, CP_N, cap) SoA
    int* parents;          // (nq, 2, cap)
    int cap;
    int nq;
    int* queue_head;
    int* team_counter;
    SceneSm scene_g;       // global-memory scene (staged to smem by each CTA)
    Con<float> con;
    ProjArgs pa;
    int W;
    float step, tol, margin;
    int flag_on;
    int max_iterations, max_connect;
    i64 budget_ns;         // 0: no time budget (deterministic); < 0: expired before the first sample
    int solo;              // 1: one team per warp (the other half-warp idles) -- latency mode
    int n_race;            // racers of a cprrtc_plan_race call (0: no race)
    int* race_flag;        // this racer's first-solution word (polled)
    int* race_peers[8];    // every racer's word (peer-mapped); the winner stores 1 to each
    // results (planner.py:488-505): the path by the solving team, status and
    // counters by the last team to leave each query
    struct QueryOut* out;  // (nq) mapped host memory
    float* paths;          // (nq, path_cap, CP_N) mapped host memory
    int* sources;          // (nq, path_cap) mapped host memory
    int* chain;            // (nq, path_cap) device scratch: path position -> node
    int path_cap;
    int pair;              // 1: two-warp teams (single queries; warp P projects, warp C certifies)
    const i64* seeds;      // (nq) Halton offsets (= QueryState.seed_offset; read before init completes)
    // single query in pair mode: the FP64 endpoint checks run on the first
    // two teams' certifier warps (no cp_check_kernel launch in the graph)
    int chk_in_kernel;
    SetupArgs chk;
};

struct QueryOut {
    int status;            // 0 Solved, 1 TimedOut, 2 IterLimit, 3 tree full, 4 path overflow,
                           // 5 stopped by another racer, -1 setup
    int setup_code;
    int path_len;
    int n_nodes[2];
    int pad;
    double device_ms;
    double total_ms;       // init -> the last team out (globaltimer)
    u64 stats[ST_NSTAT];
    // completion words (the call's sequence number, from the input block):
    // written last, behind a system-scope fence, by the query's finalizer and
    // by the endpoint check; the host polls them instead of the graph's event
    unsigned done_seq, chk_seq;
};

#endif
