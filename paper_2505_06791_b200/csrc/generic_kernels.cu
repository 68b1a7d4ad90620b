// generic_kernels.cu -- robot-independent kernels compiled ahead of time by
// nvcc for sm_100a (everything robot-specific is NVRTC, see runtime.cpp).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace cprrtc {

// sphere_aabb_clearance / sphere_sphere_clearance (maniplan/_kernels/pure.py:40-69), FP64.
__global__ void clearance_kernel(int B, int kind, const double* __restrict__ a, const double* __restrict__ b,
                                 double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const double* s = a + 4 * (size_t)i;
    double cx = s[0], cy = s[1], cz = s[2], r = s[3];
    if (kind == 0) {
        const double* bx = b + 6 * (size_t)i;
        double d2 = 0.0, t;
        if (cx < bx[0]) { t = bx[0] - cx; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        else if (cx > bx[3]) { t = cx - bx[3]; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        if (cy < bx[1]) { t = bx[1] - cy; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        else if (cy > bx[4]) { t = cy - bx[4]; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        if (cz < bx[2]) { t = bx[2] - cz; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        else if (cz > bx[5]) { t = cz - bx[5]; d2 = __dadd_rn(d2, __dmul_rn(t, t)); }
        out[i] = __dsub_rn(__dsqrt_rn(d2), r);
    } else {
        const double* o = b + 4 * (size_t)i;
        double dx = cx - o[0], dy = cy - o[1], dz = cz - o[2];
        double ss = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        out[i] = __dsub_rn(__dsqrt_rn(ss), __dadd_rn(r, o[3]));
    }
}

// J^T (J J^T + lam^2 I)^-1 e by Cholesky (pure.py:437-480), FP64, m <= 5, n <= 32.
__global__ void damped_step_kernel(int B, int m, int n, const double* __restrict__ J, const double* __restrict__ e,
                                   double lam, double* __restrict__ step, int32_t* __restrict__ ok) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double* Jb = J + (size_t)b * m * n;
    const double* eb = e + (size_t)b * m;
    double L[5][5], y[5], z[5];
    int good = 1;
    for (int i = 0; i < m && good; i++)
        for (int j = 0; j <= i; j++) {
            double acc = 0.0;
            for (int k = 0; k < n; k++) acc = __dadd_rn(acc, __dmul_rn(Jb[i * n + k], Jb[j * n + k]));
            if (i == j) acc = __dadd_rn(acc, __dmul_rn(lam, lam));
            for (int k = 0; k < j; k++) acc = __dsub_rn(acc, __dmul_rn(L[i][k], L[j][k]));
            if (i == j) {
                if (!(acc > 0.0)) { good = 0; break; }
                L[i][i] = __dsqrt_rn(acc);
            } else {
                L[i][j] = __ddiv_rn(acc, L[j][j]);
            }
        }
    ok[b] = good;
    double* sb = step + (size_t)b * n;
    if (!good) {
        for (int k = 0; k < n; k++) sb[k] = 0.0;
        return;
    }
    for (int i = 0; i < m; i++) {
        double acc = eb[i];
        for (int k = 0; k < i; k++) acc = __dsub_rn(acc, __dmul_rn(L[i][k], y[k]));
        y[i] = __ddiv_rn(acc, L[i][i]);
    }
    for (int i = m - 1; i >= 0; i--) {
        double acc = y[i];
        for (int k = i + 1; k < m; k++) acc = __dsub_rn(acc, __dmul_rn(L[k][i], z[k]));
        z[i] = __ddiv_rn(acc, L[i][i]);
    }
    for (int k = 0; k < n; k++) sb[k] = 0.0;
    for (int i = 0; i < m; i++)
        for (int k = 0; k < n; k++) sb[k] = __dadd_rn(sb[k], __dmul_rn(Jb[i * n + k], z[i]));
}

cudaError_t launch_clearance(int B, int kind, const double* a, const double* b, double* out, cudaStream_t st) {
    clearance_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, kind, a, b, out);
    return cudaGetLastError();
}

cudaError_t launch_damped_step(int B, int m, int n, const double* J, const double* e, double lam, double* step,
                               int32_t* ok, cudaStream_t st) {
    damped_step_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, m, n, J, e, lam, step, ok);
    return cudaGetLastError();
}

}  // namespace cprrtc
