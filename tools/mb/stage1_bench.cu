// Stage-1 latency microbenchmark: one team (16 lanes) of one warp evaluates
// cp_stage1 back to back (xn fed back as xt), clock64-timed.  Built against
// the dumped NVRTC translation unit (tools/dump_src.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o stage1_bench \
//        -DTU='"../../cprrtc-plan-g16-k0-o1.cu"' stage1_bench.cu
#include TU
#include <cstdio>

extern "C" __global__ void stage1_bench(int iters, long long* cyc, float* out) {
    ProjArgs pa;
    pa.alpha = 0.1f; pa.lam = 1e-3f; pa.tau_task = 0.01f; pa.tau_task_dev = 0.01f * 0.999f - 2e-6f;
    pa.tau_sm_fixed = 0.3f; pa.max_iters = 128; pa.mode = 0;
    const int lane = threadIdx.x & 31;
    float xt[CP_N], xp[CP_N], xn[CP_N];
    const float q0[7] = {0.1f, -0.4f, 0.05f, -2.2f, 0.02f, 1.9f, 0.8f};
    for (int k = 0; k < CP_N; k++) { xt[k] = q0[k % 7] + 0.01f * lane; xp[k] = q0[k % 7]; }
    bool acc = false;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        acc ^= cp_stage1(pa, xt, xp, 0.3f, xn);
        for (int k = 0; k < CP_N; k++) xt[k] = xn[k];
    }
    long long t1 = clock64();
    if (lane == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = xt[0] + (acc ? 1.f : 0.f);
}

extern "C" __global__ void part_bench(int iters, int part, long long* cyc, float* out) {
    const int lane = threadIdx.x & 31;
    float q[CP_N];
    const float q0[7] = {0.1f, -0.4f, 0.05f, -2.2f, 0.02f, 1.9f, 0.8f};
    for (int k = 0; k < CP_N; k++) q[k] = q0[k % 7] + 0.01f * lane;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (part == 0) {          // FK only (every joint angle depends on the last EE pose)
            float R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
            cp_fk<float>(q, R, P, AX, OR, SPH);
            const float d = 1e-6f * (P[3 * CP_EE] + R[9 * CP_EE]);
            for (int k = 0; k < CP_N; k++) q[k] += d;
        } else if (part >= 3) {   // FK + quaternion (3), + rotation vector (4), + SO(3) rate (5)
            float R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
            cp_fk<float>(q, R, P, AX, OR, SPH);
            float qe[4];
            cp_quat<float>(R + 9 * CP_EE, qe);
            float d = qe[0] + qe[1];
            if (part >= 4) {
                float v[3];
                const float k = cp_relrot(cp_conf, qe, v);
                d = k * v[0];
                if (part >= 5) {
                    float A9[9];
                    cp_so3_rate<float>(k * v[0], k * v[1], k * v[2], A9);
                    d = A9[0] + A9[4] + A9[8];
                }
            }
            d *= 1e-6f;
            for (int k = 0; k < CP_N; k++) q[k] += d;
        } else if (part == 1) {   // FK + quaternion + task error + Jacobian
            float e[CP_M], J[CP_M][CP_N];
            cp_err_jac<float>(cp_conf, q, e, J);
            float d = 0.f;
            for (int k = 0; k < CP_N; k++) d += J[CP_M - 1][k];
            d = 1e-6f * (d + e[0]);
            for (int k = 0; k < CP_N; k++) q[k] += d;
        } else {                  // damped least-squares step alone on a fixed J
            float e[CP_M], J[CP_M][CP_N], g[CP_N];
            for (int i2 = 0; i2 < CP_M; i2++) {
                e[i2] = 0.01f * q[i2 % CP_N];
                for (int k = 0; k < CP_N; k++) J[i2][k] = 0.1f * (i2 + 1) + 0.05f * k + 1e-3f * q[k];
            }
#if CP_M == 4
            cp_damped_f4(J, e, 1e-3f, g);
#else
            cp_damped_f<CP_M>(J, e, 1e-3f, g);
#endif
            for (int k = 0; k < CP_N; k++) q[k] += 1e-6f * g[k];
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = q[0];
}

// Halton sample (FP64, bit-exact with the reference) latency, lane k = joint k
extern "C" __global__ void halton_bench(int iters, long long seed, long long* cyc, double* out) {
    const int lane = threadIdx.x;
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (lane < CP_N) acc += cp_halton((i64)(500 + i) + seed + (acc > 1e300 ? 1 : 0), lane);
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = acc;
}

// one Alg. 1 projection of a 16-waypoint segment from an on-manifold start
// toward a point 0.5 rad away (the planner's P1), repeated
extern "C" __global__ void proj_bench(int reps, long long* cyc, int* iters_out, const int* stop, float span = 1.f) {
    __shared__ float seg[CP_G][CP_NP];
    __shared__ __align__(16) int pslot[12];
    Team tm;
    const float qa[7] = {-0.07434654f, 0.54688579f, 2.74340846f, -2.4217312f, -0.20725576f, 1.89866585f, 2.79144559f};
    const float dq[7] = {0.25f, -0.2f, -0.15f, 0.2f, -0.15f, 0.1f, -0.2f};
    ProjArgs pa;
    pa.alpha = 0.1f; pa.lam = 1e-3f; pa.tau_task = 0.01f; pa.tau_task_dev = 0.01f * 0.999f - 2e-6f;
    pa.tau_sm_fixed = 0.f; pa.max_iters = 128; pa.mode = 0;
    long long total = 0;
    int its = 0;
    for (int r = 0; r < reps; r++) {
        const int t = tm.lane;
        for (int k = 0; k < CP_N; k++) seg[t][k] = qa[k] + span * (float)t / 15.f * dq[k];
        __syncwarp();
        int it, pr;
        long long t0 = clock64();
        bool okp = cp_project(tm, seg, 16, pa, &it, &pr, nullptr, nullptr, nullptr, stop, stop ? pslot : nullptr);
        long long t1 = clock64();
        if (r == 0 && threadIdx.x == 0) printf("ok %d iters %d prog %d err0 %g\n", (int)okp, it, pr, cp_err_norm(seg[0]));
        total += t1 - t0;
        its += it;
    }
    if (threadIdx.x == 0) { cyc[0] = total; iters_out[0] = its; }
}

int main() {
    Con<float> c{};
    c.anchor[2] = 1.f; c.offset = 0.6f;
    c.qf[0] = 0.f; c.qf[1] = 1.f; c.qf[2] = 0.f; c.qf[3] = 0.f;
    float rft[9] = {1, 0, 0, 0, -1, 0, 0, 0, -1};
    for (int i = 0; i < 9; i++) c.rft[i] = rft[i];
    c.weight = 0.5f;
    cudaMemcpyToSymbol(cp_conf, &c, sizeof c);
    long long* cyc; float* out; long long h;
    cudaMalloc(&cyc, 8); cudaMalloc(&out, 4096);
    const int it = 2000;
    stage1_bench<<<1, 16>>>(it, cyc, out);
    stage1_bench<<<1, 16>>>(it, cyc, out);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("stage1: %.0f cycles per evaluation (1 warp, 16 lanes)\n", (double)h / it);
    for (int part = 0; part < 6; part++) {
        part_bench<<<1, 16>>>(it, part, cyc, out);
        part_bench<<<1, 16>>>(it, part, cyc, out);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const char* nm[6] = {"fk", "fk+err+jac", "damped", "fk+quat", "fk+quat+rotvec", "fk+quat+rotvec+so3"};
        printf("part %s: %.0f cycles\n", nm[part], (double)h / it);
    }
    {
        double* dout; cudaMalloc(&dout, 256);
        for (long long seed : {0LL, 10000LL, 1000000LL}) {
            halton_bench<<<1, 16>>>(200, seed, cyc, dout);
            halton_bench<<<1, 16>>>(200, seed, cyc, dout);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("halton (seed_offset %lld): %.0f cycles per sample\n", seed, (double)h / 200);
        }
    }
    int* its; int hi;
    cudaMalloc(&its, 4);
    int* stop;
    cudaMalloc(&stop, 1 << 20);
    cudaMemset(stop, 0, 1 << 20);
    for (int v = 0; v < 3; v++) {
        const int* sp = v == 0 ? nullptr : stop + (v - 1) * 4096;
        proj_bench<<<1, 16>>>(20, cyc, its, sp);
        proj_bench<<<1, 16>>>(20, cyc, its, sp);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hi, its, 4, cudaMemcpyDeviceToHost);
        printf("projection (stop word %s): %d iterations per call, %.0f cycles per iteration\n",
               v == 0 ? "none" : (v == 1 ? "A" : "B"), hi / 20, (double)h / hi);
    }
    // short motions (the certifier's re-projections converge in a few
    // iterations): the per-call fixed cost shows
    for (float span : {0.05f, 0.01f}) {
        proj_bench<<<1, 16>>>(20, cyc, its, stop, span);
        proj_bench<<<1, 16>>>(20, cyc, its, stop, span);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hi, its, 4, cudaMemcpyDeviceToHost);
        printf("short projection (span %.2f): %d iterations per call, %.0f cycles per call\n", span, hi / 20,
               (double)h / 20);
    }
    return 0;
}
