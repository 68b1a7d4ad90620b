// cprrtc_device.cuh -- B200 (sm_100a) device code of the cpRRTC planner.
//
// Compiled at run time by NVRTC (csrc/runtime.cpp) after a generated prelude
// that supplies the robot (unrolled FK `cp_fk`, limits, radii, self pairs; see
// csrc/codegen.cpp) and the module configuration:
//   CP_G       team width in lanes (16 or 32): one team = one extension
//   CP_KIND    0 plane / 1 line position constraint     (compile-time)
//   CP_ORIENT  1 if the EE orientation is locked         (compile-time)
//   CP_NTHREADS threads per CTA of the persistent planner
//
// Execution model: a team of CP_G lanes of one warp
// owns one tree extension at a time -- lane t holds waypoint t of the motion
// (the paper's "one thread per waypoint").  Alg. 1's barriers
// become a shuffle of row t-1 and a ballot, stage 2's prefix scan the ballot,
// and the paper's shared-memory collision flag a team vote per
// chunk of primitives.  Single queries pair two warps per team (warp P
// projects, warp C certifies one motion behind, mbarrier hand-offs).
// Obstacles are staged once per CTA in shared memory; trees are SoA float
// arrays in HBM with atomic append.
//
// Every function cites the reference function it replaces
// (maniplan/..., /root/reference/pkg/src/).

#ifndef CP_G
#error "CP_G must be defined by the runtime prelude"
#endif

#define CP_M ((CP_KIND == 0 ? 1 : 2) + (CP_ORIENT ? 3 : 0))
// packed box test clamp: 1 = FMNMX on the ALU pipe (vs r^2), 0 = t + |t| on
// the FP32 pipe (squared sum 4x, vs 4 r^2).  r2 A/B on the 999-box CC kernel:
// 2.18 vs 2.10 T checks/s (with the sphere pairs pre-packed, the FP32 pipe is
// the tighter one, so the clamp goes to the ALU)
#ifndef CP_CC_CLAMP_ALU
#define CP_CC_CLAMP_ALU 1
#endif
#define CP_CC_RSCALE (CP_CC_CLAMP_ALU ? 1.f : 4.f)
#define CP_NP ((CP_N % 2) ? CP_N : (CP_N + 1))   // odd row pitch: no bank conflicts
#define CP_CHUNK 8
#define CP_VOTE 4                    // lockstep CC: early-exit vote every CP_VOTE chunks
#ifndef CP_ROOT_FIRST
#define CP_ROOT_FIRST 1              // single query: the first extension's nearest node is the root
#endif
#ifndef CP_ROOT_FIRST_CONNECT
#define CP_ROOT_FIRST_CONNECT 0      // single query: round 0's connect starts at tree b's root too (A/B knob)
#endif
#ifndef CP_SPEC_JUNC
#define CP_SPEC_JUNC 1               // pair mode: the junction runs while C certifies the meeting motion
#endif
#ifndef CP_NN_PAIRS
#define CP_NN_PAIRS 1                // planner NN: two chunks per L2 round trip
#endif
#define CP_BCH (2 + 2 * CP_CHUNK)   // float4s per box chunk of the clustered scene
#define CP_SCH (2 + CP_CHUNK)       // float4s per sphere chunk
#define CP_INTMAX 0x7fffffff
#define CP_PATH_CAP 4096


__device__ __forceinline__ float cp_inf() { return __int_as_float(0x7f800000); }
__device__ __forceinline__ u64 cp_clock_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ float4 cp_ldcg4(const float* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ int cp_ldvol(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ unsigned long long cp_ldvol64(const unsigned long long* p) { return *(const volatile unsigned long long*)p; }
template <class T> __device__ __forceinline__ bool cp_finite(T x) { return isfinite(x); }

// ---------------------------------------------------------------------------
// team = CP_G lanes of a warp
// ---------------------------------------------------------------------------
struct Team {
    unsigned lane, base, mask;
    __device__ Team() {
        unsigned l = threadIdx.x & 31u;
        lane = l % CP_G;
        base = l - lane;
        mask = (CP_G == 32) ? 0xffffffffu : (0xffffu << base);
    }
    __device__ __forceinline__ unsigned ballot(bool p) const {
        return __ballot_sync(mask, p) >> base;
    }
    __device__ __forceinline__ bool any(bool p) const { return ballot(p) != 0u; }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ int bcast(int v, int src) const { return __shfl_sync(mask, v, src, CP_G); }
    __device__ __forceinline__ float bcastf(float v, int src) const { return __shfl_sync(mask, v, src, CP_G); }
    __device__ __forceinline__ float sum(float v) const {
#pragma unroll
        for (int o = CP_G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, CP_G);
        return v;
    }
    __device__ __forceinline__ float maxf(float v) const {
#pragma unroll
        for (int o = CP_G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(mask, v, o, CP_G));
        return v;
    }
    // lexicographic (key, idx) minimum over the team
    __device__ __forceinline__ void argmin(float& key, int& idx) const {
#pragma unroll
        for (int o = CP_G / 2; o > 0; o >>= 1) {
            float k2 = __shfl_xor_sync(mask, key, o, CP_G);
            int i2 = __shfl_xor_sync(mask, idx, o, CP_G);
            if (k2 < key || (k2 == key && i2 < idx)) { key = k2; idx = i2; }
        }
    }
    __device__ __forceinline__ void argmin_i(int& key, int& idx) const {
#pragma unroll
        for (int o = CP_G / 2; o > 0; o >>= 1) {
            int k2 = __shfl_xor_sync(mask, key, o, CP_G);
            int i2 = __shfl_xor_sync(mask, idx, o, CP_G);
            if (k2 < key || (k2 == key && i2 < idx)) { key = k2; idx = i2; }
        }
    }
};

// ---------------------------------------------------------------------------
// constraint (packed layout of maniplan/constraints.py:123-176)
// ---------------------------------------------------------------------------

// Division traits.  FP64 (parity / setup paths) keeps the reference's exact
// operations; FP32 (planner) divides by a diagonal / pivot through one
// reciprocal (MUFU) and multiplies.
template <class T> struct CpDiv {
    static __device__ __forceinline__ T piv(T x) { return x; }           // stored pivot
    static __device__ __forceinline__ T div(T a, T p) { return a / p; }  // a / pivot
    static __device__ __forceinline__ T sqrt_piv(T x) { return sqrt(x); }
    // s = 2 sqrt(x) and its pivot
    static __device__ __forceinline__ T twice_sqrt(T x, T& p) { T s = sqrt(x) * T(2); p = s; return s; }
};
template <> struct CpDiv<float> {
    static __device__ __forceinline__ float piv(float x) { return __fdividef(1.f, x); }
    static __device__ __forceinline__ float div(float a, float p) { return a * p; }
    static __device__ __forceinline__ float sqrt_piv(float x) { return rsqrtf(x); }
    // one MUFU.RSQ gives both 2 sqrt(x) and 1 / (2 sqrt(x))
    static __device__ __forceinline__ float twice_sqrt(float x, float& p) {
        const float r = rsqrtf(x);
        p = 0.5f * r;
        return 2.f * (x * r);
    }
};

// rotation -> quaternion, w >= 0 (maniplan/_kernels/pure.py:130-159)
template <class T>
__device__ __forceinline__ void cp_quat(const T* r, T* q) {
    T w, x, y, z, s;
    T tr = (r[0] + r[4]) + r[8];
    if (tr > T(0)) {
        T is;
        s = CpDiv<T>::twice_sqrt(tr + T(1), is);
        w = T(0.25) * s; x = CpDiv<T>::div(r[7] - r[5], is); y = CpDiv<T>::div(r[2] - r[6], is);
        z = CpDiv<T>::div(r[3] - r[1], is);
    } else if (r[0] > r[4] && r[0] > r[8]) {
        T is;
        s = CpDiv<T>::twice_sqrt(((T(1) + r[0]) - r[4]) - r[8], is);
        w = CpDiv<T>::div(r[7] - r[5], is); x = T(0.25) * s; y = CpDiv<T>::div(r[1] + r[3], is);
        z = CpDiv<T>::div(r[2] + r[6], is);
    } else if (r[4] > r[8]) {
        T is;
        s = CpDiv<T>::twice_sqrt(((T(1) + r[4]) - r[0]) - r[8], is);
        w = CpDiv<T>::div(r[2] - r[6], is); x = CpDiv<T>::div(r[1] + r[3], is); y = T(0.25) * s;
        z = CpDiv<T>::div(r[5] + r[7], is);
    } else {
        T is;
        s = CpDiv<T>::twice_sqrt(((T(1) + r[8]) - r[0]) - r[4], is);
        w = CpDiv<T>::div(r[3] - r[1], is); x = CpDiv<T>::div(r[2] + r[6], is);
        y = CpDiv<T>::div(r[5] + r[7], is); z = T(0.25) * s;
    }
    if (w < T(0)) { w = -w; x = -x; y = -y; z = -z; }
    q[0] = w; q[1] = x; q[2] = y; q[3] = z;
}

// rotation-vector scale k = 2 atan2(vn, rw) / vn of a unit quaternion with
// rw, vn >= 0, from s2 = vn^2 (pure.py:338-344).  FP32: atan(x)/x on x in [0, 1] as a
// degree-8 polynomial in x^2 (max relative error 9e-8, fitted for this file),
// with the reflection atan(x) = pi/2 - atan(1/x) above 1.
template <class T> __device__ __forceinline__ T cp_rotscale(T s2, T rw) {
    const T vn = sqrt(s2);
    return vn < T(1e-12) ? T(2) : T(2) * atan2(vn, rw) / vn;
}
template <> __device__ __forceinline__ float cp_rotscale<float>(float s2, float rw) {
    // s2 = |v|^2: 1/|v| and 1/w are independent MUFU ops (no sqrt -> divide chain)
    const float ivn = rsqrtf(s2), irw = __fdividef(1.f, rw);
    const float vn = s2 * ivn;
    if (!(s2 >= 1e-24f)) return 2.f;   // |v| < 1e-12 (pure.py:343)
    const bool sw = vn > rw;
    const float x = sw ? rw * ivn : vn * irw;
    const float u = x * x;
    float p = 0.0028531861025840044f;
    p = fmaf(p, u, -0.016082055866718292f);
    p = fmaf(p, u, 0.042713798582553864f);
    p = fmaf(p, u, -0.07506226748228073f);
    p = fmaf(p, u, 0.1064186692237854f);
    p = fmaf(p, u, -0.14203891158103943f);
    p = fmaf(p, u, 0.19992651045322418f);
    p = fmaf(p, u, -0.33333075046539307f);
    p = fmaf(p, u, 1.0f);
    return sw ? 2.f * fmaf(-x, p, 1.5707963267948966f) * ivn : 2.f * p * irw;
}

// q_fixed^-1 * q_ee as a rotation vector k*v (pure.py:328-344)
template <class T>
__device__ __forceinline__ T cp_relrot(const Con<T>& c, const T* qe, T* v) {
    T aw = c.qf[0], ax = -c.qf[1], ay = -c.qf[2], az = -c.qf[3];
    T rw = ((aw * qe[0] - ax * qe[1]) - ay * qe[2]) - az * qe[3];
    T rx = ((aw * qe[1] + ax * qe[0]) + ay * qe[3]) - az * qe[2];
    T ry = ((aw * qe[2] - ax * qe[3]) + ay * qe[0]) + az * qe[1];
    T rz = ((aw * qe[3] + ax * qe[2]) - ay * qe[1]) + az * qe[0];
    if (rw < T(0)) { rw = -rw; rx = -rx; ry = -ry; rz = -rz; }
    v[0] = rx; v[1] = ry; v[2] = rz;
    return cp_rotscale<T>((rx * rx + ry * ry) + rz * rz, rw);
}

// Rotation vector of q_fixed^-1 q_ee straight from the EE rotation matrix
// (pure.py:328-344 goes through the quaternion).  Generic / FP64: the
// reference's quaternion route.  FP32 planner: the matrix logarithm of
// M = R_fixed^T R_ee -- cos(theta) = (tr M - 1)/2, sin(theta) axis = vee(M - M^T)/2,
// theta = atan2(sin, cos) with the polynomial atan -- which is the same
// rotation vector without the quaternion's branches and square roots; near
// theta = pi (cos < -0.7) the skew part is ill-conditioned and the axis comes
// from the symmetric part instead (both evaluated, selected: no branch).
template <class T>
__device__ __forceinline__ void cp_orient_rotvec(const Con<T>& c, const T* Ree, T* rv) {
    T qe[4], v[3];
    cp_quat<T>(Ree, qe);
    const T k = cp_relrot(c, qe, v);
    rv[0] = k * v[0]; rv[1] = k * v[1]; rv[2] = k * v[2];
}
template <>
__device__ __forceinline__ void cp_orient_rotvec<float>(const Con<float>& c, const float* R, float* rv) {
    const float* f = c.rft;   // R_fixed^T, row-major
    auto m = [&](int i, int j) { return fmaf(f[3 * i], R[j], fmaf(f[3 * i + 1], R[3 + j], f[3 * i + 2] * R[6 + j])); };
    const float m00 = m(0, 0), m11 = m(1, 1), m22 = m(2, 2);
    const float m01 = m(0, 1), m10 = m(1, 0), m02 = m(0, 2), m20 = m(2, 0), m12 = m(1, 2), m21 = m(2, 1);
    const float vx = 0.5f * (m21 - m12), vy = 0.5f * (m02 - m20), vz = 0.5f * (m10 - m01);
    const float cth = 0.5f * ((m00 + m11) + m22 - 1.f);
    const float s2 = fmaf(vx, vx, fmaf(vy, vy, vz * vz));
    const float ivn = rsqrtf(s2), vn = s2 * ivn, ac = fabsf(cth), iac = __fdividef(1.f, ac);
    // theta = atan2(vn, cth) through atan(x) on x in [0, 1]
    const bool sw = vn > ac;
    const float x = sw ? ac * ivn : vn * iac;
    const float u = x * x;
    float p = 0.0028531861025840044f;
    p = fmaf(p, u, -0.016082055866718292f);
    p = fmaf(p, u, 0.042713798582553864f);
    p = fmaf(p, u, -0.07506226748228073f);
    p = fmaf(p, u, 0.1064186692237854f);
    p = fmaf(p, u, -0.14203891158103943f);
    p = fmaf(p, u, 0.19992651045322418f);
    p = fmaf(p, u, -0.33333075046539307f);
    p = fmaf(p, u, 1.0f);
    const float at = x * p;                                   // atan(x)
    const float half = sw ? 1.5707963267948966f - at : at;   // atan2(vn, |cth|)
    const float th = cth >= 0.f ? half : 3.14159265358979f - half;
    // well-conditioned regime: rotation vector = theta / sin(theta) * v
    float sc = sw ? th * ivn : (cth >= 0.f ? p * iac : th * ivn);
    sc = s2 >= 1e-24f ? sc : 1.f;
    // near theta = pi (cth < -0.7) the skew part vanishes: the axis comes from
    // the symmetric part instead, B = (M + M^T)/2 - c I = (1 - c) a a^T: the
    // column of the largest diagonal entry k gives a = B[:, k] / sqrt((1-c) B_kk)
    // (one well-conditioned square root), its sign from the skew part
    // (sin theta > 0).  Both regimes are evaluated and selected (no branch).
    const float d0 = m00 - cth, d1 = m11 - cth, d2 = m22 - cth;
    const float s01 = 0.5f * (m01 + m10), s02 = 0.5f * (m02 + m20), s12 = 0.5f * (m12 + m21);
    const bool k0 = d0 >= d1 && d0 >= d2, k1 = !k0 && d1 >= d2;
    const float dk = k0 ? d0 : (k1 ? d1 : d2);
    const float nk = rsqrtf(fmaxf((1.f - cth) * dk, 1e-30f));
    float b0 = (k0 ? d0 : (k1 ? s01 : s02)) * nk;
    float b1 = (k0 ? s01 : (k1 ? d1 : s12)) * nk;
    float b2 = (k0 ? s02 : (k1 ? s12 : d2)) * nk;
    const float sg = fmaf(b0, vx, fmaf(b1, vy, b2 * vz)) < 0.f ? -th : th;
    const bool nearpi = cth < -0.7f;
    rv[0] = nearpi ? sg * b0 : sc * vx;
    rv[1] = nearpi ? sg * b1 : sc * vy;
    rv[2] = nearpi ? sg * b2 : sc * vz;
}

// task error rows at a pose (pure.py:312-345): position rows, then (locked
// orientation) the weighted rotation vector k*v of q_fixed^-1 q_ee
template <class T>
__device__ __forceinline__ void cp_task_err_kv(const Con<T>& c, const T* p, T k, const T* v, T* e) {
    int m = 0;
#if CP_KIND == 0
    e[m++] = ((c.anchor[0] * p[0] + c.anchor[1] * p[1]) + c.anchor[2] * p[2]) - c.offset;
#else
    T dx = p[0] - c.anchor[0], dy = p[1] - c.anchor[1], dz = p[2] - c.anchor[2];
    e[m++] = (c.b1[0] * dx + c.b1[1] * dy) + c.b1[2] * dz;
    e[m++] = (c.b2[0] * dx + c.b2[1] * dy) + c.b2[2] * dz;
#endif
#if CP_ORIENT
    e[m++] = c.weight * (k * v[0]);
    e[m++] = c.weight * (k * v[1]);
    e[m++] = c.weight * (k * v[2]);
#endif
    (void)k; (void)v;
}
template <class T>
__device__ __forceinline__ void cp_task_err(const Con<T>& c, const T* p, const T* qe, T* e) {
    T v[3] = {T(0), T(0), T(0)}, k = T(0);
#if CP_ORIENT
    k = cp_relrot(c, qe, v);
#endif
    cp_task_err_kv<T>(c, p, k, v, e);
    (void)qe;
}

// c2(theta) = 1/theta^2 - (1 + cos theta) / (2 theta sin theta) of the inverse
// left Jacobian (pure.py:352-358).  FP32: a polynomial in theta^2 (the closed
// form cancels catastrophically in FP32 for small theta).
template <class T> __device__ __forceinline__ T cp_so3_c2(T t2) {
    if (t2 < T(1e-8)) return T(1.0 / 12.0) + t2 / T(720);
    T th = sqrt(t2), s, co;
    sincos(th, &s, &co);
    return T(1) / t2 - (T(1) + co) / ((T(2) * th) * s);
}
template <> __device__ __forceinline__ float cp_so3_c2<float>(float t2) {
    // minimax polynomial in t2 over [0, pi^2] (every rotation-vector angle),
    // max relative error 8e-8 in FP32: branch-free, no cancellation
    float p = 3.002027066604379e-14f;
    p = fmaf(p, t2, -1.5192574032586031e-13f);
    p = fmaf(p, t2, 1.8825586922677218e-11f);
    p = fmaf(p, t2, 4.946845155728852e-10f);
    p = fmaf(p, t2, 2.0997001470846044e-08f);
    p = fmaf(p, t2, 8.264817665804003e-07f);
    p = fmaf(p, t2, 3.306901635369286e-05f);
    p = fmaf(p, t2, 0.00138888880610466f);
    return fmaf(p, t2, 0.0833333358168602f);
}

// inverse left Jacobian of SO(3) (pure.py:348-366)
template <class T>
__device__ __forceinline__ void cp_so3_rate(T p0, T p1, T p2, T* a) {
    T t2 = (p0 * p0 + p1 * p1) + p2 * p2;
    T c2 = cp_so3_c2<T>(t2);
    T h0 = T(0.5) * p0, h1 = T(0.5) * p1, h2 = T(0.5) * p2;
    T c01 = c2 * (p0 * p1), c02 = c2 * (p0 * p2), c12 = c2 * (p1 * p2);
    a[0] = T(1) - c2 * (p1 * p1 + p2 * p2); a[1] = h2 + c01; a[2] = c02 - h1;
    a[3] = c01 - h2; a[4] = T(1) - c2 * (p0 * p0 + p2 * p2); a[5] = h0 + c12;
    a[6] = h1 + c02; a[7] = c12 - h0; a[8] = T(1) - c2 * (p0 * p0 + p1 * p1);
}

// (e, J) at q from one FK pass (pure.py:369-427).  Returns the EE pose too.
template <class T>
__device__ __forceinline__ void cp_err_jac(const Con<T>& c, const T* q, T* e, T (*J)[CP_N]) {
    T R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
    cp_fk<T>(q, R, P, AX, OR, SPH);
    const T* pe = P + 3 * CP_EE;
#if CP_ORIENT
    T rv[3], A[9], Mo[9];
    cp_orient_rotvec<T>(c, R + 9 * CP_EE, rv);   // once: shared by the error rows and the Jacobian
    cp_task_err_kv<T>(c, pe, T(1), rv, e);
    cp_so3_rate<T>(rv[0], rv[1], rv[2], A);
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            Mo[3 * i + j] = c.weight * ((A[3 * i] * c.rft[j] + A[3 * i + 1] * c.rft[3 + j]) + A[3 * i + 2] * c.rft[6 + j]);
#else
    cp_task_err_kv<T>(c, pe, T(0), pe, e);
#endif
#pragma unroll
    for (int j = 0; j < CP_N; j++) {
        const T* a = AX + 3 * j;
        T l0, l1, l2;
        if (cp_jtype(j) == 0) {
            T rx = pe[0] - OR[3 * j], ry = pe[1] - OR[3 * j + 1], rz = pe[2] - OR[3 * j + 2];
            l0 = a[1] * rz - a[2] * ry; l1 = a[2] * rx - a[0] * rz; l2 = a[0] * ry - a[1] * rx;
        } else {
            l0 = a[0]; l1 = a[1]; l2 = a[2];
        }
        int r = 0;
#if CP_KIND == 0
        J[r++][j] = (c.anchor[0] * l0 + c.anchor[1] * l1) + c.anchor[2] * l2;
#else
        J[r++][j] = (c.b1[0] * l0 + c.b1[1] * l1) + c.b1[2] * l2;
        J[r++][j] = (c.b2[0] * l0 + c.b2[1] * l1) + c.b2[2] * l2;
#endif
#if CP_ORIENT
        if (cp_jtype(j) == 0) {
#pragma unroll
            for (int i = 0; i < 3; i++) J[r + i][j] = (Mo[3 * i] * a[0] + Mo[3 * i + 1] * a[1]) + Mo[3 * i + 2] * a[2];
        } else {
#pragma unroll
            for (int i = 0; i < 3; i++) J[r + i][j] = T(0);
        }
#endif
        (void)r;
    }
}

// J^T (J J^T + lam^2 I)^-1 e by Cholesky; false when not SPD (pure.py:437-480)
template <class T, int M>
__device__ __forceinline__ bool cp_damped(const T (*J)[CP_N], const T* e, T lam, T* step) {
    T L[M][M], y[M], z[M];
#pragma unroll
    for (int i = 0; i < M; i++)
#pragma unroll
        for (int j = 0; j <= i; j++) {
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < CP_N; k++) acc += J[i][k] * J[j][k];
            if (i == j) acc += lam * lam;
#pragma unroll
            for (int k = 0; k < j; k++) acc -= L[i][k] * L[j][k];
            if (i == j) {
                if (!(acc > T(0))) return false;
                L[i][i] = CpDiv<T>::sqrt_piv(acc);   // FP32 holds 1 / L_ii
            } else {
                L[i][j] = CpDiv<T>::div(acc, L[j][j]);
            }
        }
#pragma unroll
    for (int i = 0; i < M; i++) {
        T acc = e[i];
#pragma unroll
        for (int k = 0; k < i; k++) acc -= L[i][k] * y[k];
        y[i] = CpDiv<T>::div(acc, L[i][i]);
    }
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
        T acc = y[i];
#pragma unroll
        for (int k = i + 1; k < M; k++) acc -= L[k][i] * z[k];
        z[i] = CpDiv<T>::div(acc, L[i][i]);
    }
#pragma unroll
    for (int k = 0; k < CP_N; k++) {
        T acc = T(0);
#pragma unroll
        for (int i = 0; i < M; i++) acc += J[i][k] * z[i];
        step[k] = acc;
    }
    return true;
}

// Packed FP32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2: two FP32 lanes per
// instruction on a 64-bit register pair; a scalar operand is broadcast by
// packing it twice, which ptxas turns into a .F32 operand).
typedef unsigned long long cp_f2;
__device__ __forceinline__ cp_f2 cp_pk(float a, float b) {
    cp_f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void cp_upk(cp_f2 r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ cp_f2 cp_sub2(cp_f2 a, cp_f2 b) {
    cp_f2 r;
    asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cp_f2 cp_add2(cp_f2 a, cp_f2 b) {
    cp_f2 r;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cp_f2 cp_mul2(cp_f2 a, cp_f2 b) {
    cp_f2 r;
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cp_f2 cp_fma2(cp_f2 a, cp_f2 b, cp_f2 c) {
    cp_f2 r;
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// FP32 planner variant of cp_damped without early returns: a non-positive
// (or NaN) pivot marks the system singular -- the caller then takes a zero
// step (pure.py:529-531) -- and the whole solve stays one basic block, so the
// scheduler can overlap its MUFU latencies with the surrounding code.
template <int M>
__device__ __forceinline__ bool cp_damped_f(const float (*J)[CP_N], const float* e, float lam, float* step) {
    float L[M][M], y[M], z[M];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < M; i++)
#pragma unroll
        for (int j = 0; j <= i; j++) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < CP_N; k++) acc = fmaf(J[i][k], J[j][k], acc);
            if (i == j) acc += lam * lam;
#pragma unroll
            for (int k = 0; k < j; k++) acc -= L[i][k] * L[j][k];
            if (i == j) {
                ok &= acc > 0.f;
                L[i][i] = rsqrtf(fmaxf(acc, 1e-30f));   // 1 / L_ii
            } else {
                L[i][j] = acc * L[j][j];
            }
        }
#pragma unroll
    for (int i = 0; i < M; i++) {
        float acc = e[i];
#pragma unroll
        for (int k = 0; k < i; k++) acc -= L[i][k] * y[k];
        y[i] = acc * L[i][i];
    }
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
        float acc = y[i];
#pragma unroll
        for (int k = i + 1; k < M; k++) acc -= L[k][i] * z[k];
        z[i] = acc * L[i][i];
    }
#pragma unroll
    for (int k = 0; k < CP_N; k++) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < M; i++) acc = fmaf(J[i][k], z[i], acc);
        step[k] = ok ? acc : 0.f;
    }
    return ok;
}

// FP32 damped step for the plane + orientation task (m = 4) by 2x2 block
// elimination instead of the Cholesky chain: A = J J^T + lam^2 I =
// [[P, Q], [Q^T, S]] with 2x2 blocks; P^-1 and the Schur complement
// S' = S - Q^T P^-1 Q are inverted in closed form, so the solve needs two
// dependent reciprocals instead of four dependent rsqrt pivots.  A is SPD iff
// P and S' are, which is exactly when the Cholesky of pure.py:437-480 succeeds;
// otherwise (or NaN) the step is zero (pure.py:529-531).
__device__ __forceinline__ bool cp_damped_f4(const float (*J)[CP_N], const float* e, float lam, float* step) {
    float a[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j <= i; j++) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < CP_N; k++) acc = fmaf(J[i][k], J[j][k], acc);
            a[i][j] = a[j][i] = acc;
        }
    const float l2 = lam * lam;
    a[0][0] += l2; a[1][1] += l2; a[2][2] += l2; a[3][3] += l2;
    // P^-1
    const float dp = fmaf(a[0][0], a[1][1], -a[0][1] * a[0][1]);
    const float idp = __fdividef(1.f, dp);
    const float p00 = a[1][1] * idp, p01 = -a[0][1] * idp, p11 = a[0][0] * idp;
    // X = P^-1 Q  (Q = a[0..1][2..3])
    const float x00 = fmaf(p00, a[0][2], p01 * a[1][2]), x01 = fmaf(p00, a[0][3], p01 * a[1][3]);
    const float x10 = fmaf(p01, a[0][2], p11 * a[1][2]), x11 = fmaf(p01, a[0][3], p11 * a[1][3]);
    // S' = S - Q^T X
    const float s00 = a[2][2] - fmaf(a[0][2], x00, a[1][2] * x10);
    const float s01 = a[2][3] - fmaf(a[0][2], x01, a[1][2] * x11);
    const float s11 = a[3][3] - fmaf(a[0][3], x01, a[1][3] * x11);
    const float ds = fmaf(s00, s11, -s01 * s01);
    const float ids = __fdividef(1.f, ds);
    // w = P^-1 e1; r = e2 - Q^T w; y2 = S'^-1 r; y1 = w - X y2
    const float w0 = fmaf(p00, e[0], p01 * e[1]), w1 = fmaf(p01, e[0], p11 * e[1]);
    const float r0 = e[2] - fmaf(a[0][2], w0, a[1][2] * w1);
    const float r1 = e[3] - fmaf(a[0][3], w0, a[1][3] * w1);
    const float y2 = fmaf(s11, r0, -s01 * r1) * ids, y3 = fmaf(s00, r1, -s01 * r0) * ids;
    const float y0 = w0 - fmaf(x00, y2, x01 * y3), y1 = w1 - fmaf(x10, y2, x11 * y3);
    const bool ok = a[0][0] > 0.f && dp > 0.f && s00 > 0.f && ds > 0.f;
#pragma unroll
    for (int k = 0; k < CP_N; k++) {
        const float g = fmaf(J[0][k], y0, fmaf(J[1][k], y1, fmaf(J[2][k], y2, J[3][k] * y3)));
        step[k] = ok ? g : 0.f;
    }
    return ok;
}

// The FP32 constraint of the module's current call lives in constant memory
// (written by the runtime before each launch that projects), so the hot loops
// address it as constant-bank operands instead of through a pointer.
__constant__ Con<float> cp_conf;

// One out-of-line FP32 copy of (e, J) for the cold sequential projector.
__device__ __noinline__ void cp_err_jac_f(const Con<float>& c, const float* q, float* e, float (*J)[CP_N]) {
    float qq[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) qq[k] = q[k];
    cp_err_jac<float>(c, qq, e, J);
}

// ---------------------------------------------------------------------------
// projection parameters (maniplan/projection.py:75-90), FP32 with margins
// ---------------------------------------------------------------------------

// stage 1 of Alg. 1 for one waypoint (pure.py:511-546).  Validity is judged
// at the pre-update waypoint with the device margins.
// Branch-free: a non-finite waypoint is frozen (xn = xt, invalid; pure.py:
// 524-526) by selects after the (NaN-propagating) evaluation.
// Stage 1 in two parts: A needs the waypoint alone (finiteness, task error
// norm, damped Newton step -- all but a few dozen of its instructions), B adds
// the previous waypoint (the smoothing term and the validity test).
struct Stage1A {
    float g[CP_N];   // damped step (zero if singular)
    float en2;       // squared task error
    bool fin;
};

__device__ __forceinline__ void cp_stage1a(const ProjArgs& pa, const float* xt, Stage1A& a) {
    bool fin = true;
#pragma unroll
    for (int k = 0; k < CP_N; k++) fin &= cp_finite(xt[k]);
    float e[CP_M], J[CP_M][CP_N];
    cp_err_jac<float>(cp_conf, xt, e, J);
    float en2 = 0.f;
#pragma unroll
    for (int i = 0; i < CP_M; i++) en2 = fmaf(e[i], e[i], en2);
#if CP_M == 4
    cp_damped_f4(J, e, pa.lam, a.g);         // singular -> zero step (pure.py:529-531)
#else
    cp_damped_f<CP_M>(J, e, pa.lam, a.g);   // singular -> zero step (pure.py:529-531)
#endif
    a.en2 = en2;
    a.fin = fin;
}

__device__ __forceinline__ bool cp_stage1b(const ProjArgs& pa, const Stage1A& a, const float* xt, const float* xp,
                                           float tau_sm, float* xn) {
    float d[CP_N], s2 = 0.f;
#pragma unroll
    for (int k = 0; k < CP_N; k++) { d[k] = xt[k] - xp[k]; s2 = fmaf(d[k], d[k], s2); }
    float gap = sqrtf(s2);
    float exc = fmaxf(gap - tau_sm, 0.f);
#pragma unroll
    for (int k = 0; k < CP_N; k++) xn[k] = a.fin ? xt[k] - pa.alpha * (a.g[k] + d[k] * exc) : xt[k];
    return a.fin && gap < tau_sm * 0.99999f && sqrtf(a.en2) < pa.tau_task_dev;
}

__device__ __forceinline__ bool cp_stage1(const ProjArgs& pa, const float* xt,
                                          const float* xp, float tau_sm, float* xn) {
    Stage1A a;
    cp_stage1a(pa, xt, a);
    return cp_stage1b(pa, a, xt, xp, tau_sm, xn);
}

__device__ __noinline__ float cp_err_norm(const float* q) {
    float R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
    cp_fk<float>(q, R, P, AX, OR, SPH);
    float rv[3] = {0.f, 0.f, 0.f}, e[CP_M];
#if CP_ORIENT
    cp_orient_rotvec<float>(cp_conf, R + 9 * CP_EE, rv);
#endif
    cp_task_err_kv<float>(cp_conf, P + 3 * CP_EE, 1.f, rv, e);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CP_M; i++) s += e[i] * e[i];
    return sqrtf(s);
}

// The iterations of Alg. 1 (pure.py:549-568) for the team's rows xc (lane t =
// waypoint t).  UNC: tau_task = inf, validity needs no FK (pure.py:545) and the
// update is computed only if the segment is not accepted as is.  The prefix
// update is branch-free for both modes (contiguous prefix, pure.py:564-568;
// literal-gap, pure.py:560-563); the stop word rides in bit 0 of the validity
// ballot (lane 0 holds the fixed start, never active), so the poll costs no
// extra warp collective.
//
// The poll is an asynchronous 16-byte copy of the stop word's L2 sector into
// one of two shared-memory slots of the team (cp.async.cg, one commit group
// per iteration: no register scoreboard); after stage 1 the loop reads the
// copy issued one iteration earlier, behind cp.async.wait_group 1 -- which
// never waits in practice (an iteration, ~1200 cycles, covers the L2 round
// trip), wherever ptxas places it.  A stop is seen one iteration late, and
// not in a projection's first iteration: the slots alternate across
// projections (the parity persists in the workspace), so a projection starts
// with neither a prologue poll nor a wait for the previous one's last poll
// (r1: ~1 L2 round trip per call, which short re-projections felt).  r1
// (B200): a plain load cost ~300 cycles per iteration of ~1500 (ptxas turned
// its value into a predicate right after issue, stalling on the round trip),
// and a same-iteration cp.async.wait_all was hoisted the same way.
template <bool UNC, bool TRACE>
__device__ __forceinline__ void cp_alg1_loop(const Team tm, int W, const ProjArgs& pa, float tau_sm,
                                             float* xc, int& prog, int& iters, bool& ok, bool& aborted,
                                             unsigned& s1, const int* stop_flag, int* pslot,
                                             float* trace, int* trace_prog) {
    const int t = (int)tm.lane;
    const bool row = t < W;
    const unsigned full = (W >= 32) ? 0xffffffffu : ((1u << W) - 1u);
    // lane 0 polls (r1 A/B: all 16 lanes loading the word cost 5 %); the
    // issue is predicated and the wait + read run on every lane, so the loop
    // body stays one basic block (a branch around either cost ~100 cycles)
    const bool poll = stop_flag && pslot && t == 0;
    const unsigned long long sbase = (unsigned long long)stop_flag & ~15ull;
    const unsigned slot = pslot ? (unsigned)__cvta_generic_to_shared(pslot) : 0u;   // 2 x 16 B slots
    const unsigned soff = (unsigned)((unsigned long long)stop_flag - sbase);
    unsigned par = poll ? (unsigned)pslot[8] : 0u;   // slot of the next poll (lane 0; persists)
    const float tsm = tau_sm * 0.99999f;
    for (int it = 1; it <= pa.max_iters; it++) {
        const bool act = row && t > prog;
        const unsigned put = slot + 16u * (par & 1u), get = slot + 16u * ((par + 1u) & 1u) + soff;
        par ^= 1u;
        asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p cp.async.cg.shared.global [%0], [%1], 16; "
                     "cp.async.commit_group; }" ::"r"(put), "l"(sbase), "r"((unsigned)poll));
        float xn[CP_N], xp[CP_N];
#pragma unroll
        for (int k = 0; k < CP_N; k++) xp[k] = __shfl_up_sync(tm.mask, xc[k], 1, CP_G);
        bool valid = false, full_step = true;
        if (UNC) {
#pragma unroll
            for (int k = 0; k < CP_N; k++) xn[k] = xc[k];
            bool cheap = true;
            if (act) {
                float s2 = 0.f;
                bool fin = true;
#pragma unroll
                for (int k = 0; k < CP_N; k++) { float d = xc[k] - xp[k]; s2 += d * d; fin &= cp_finite(xc[k]); }
                cheap = fin && sqrtf(s2) < tsm;
            }
            if (!tm.any(!cheap)) { valid = act; full_step = false; }
        }
        if (!UNC || full_step) {
            // every lane evaluates (branch-free stage 1); frozen / idle lanes
            // discard the result
            const bool v = cp_stage1(pa, xc, xp, tau_sm, xn);
            valid = act && v;
            s1 += act ? 1u : 0u;   // per lane; summed over the team at the end
        }
        int sf;   // lane 0 only; no "memory" clobber (it would pin stage 1's constant-bank reads)
        asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; cp.async.wait_group 1; mov.u32 %0, 0; "
                     "@p ld.shared.b32 %0, [%1]; }" : "=r"(sf) : "r"(get), "r"((unsigned)(poll && it > 1)));
        const unsigned vm = tm.ballot(valid || sf != 0) & full;
        const unsigned hi = vm & ~((2u << prog) - 1u);              // literal-gap
        const int np1 = hi ? 31 - __clz(hi) : prog;
        const int run = __ffs(~(vm >> (prog + 1))) - 1;               // contiguous prefix
        const int np0 = min(prog + (run < 0 ? 32 : run), W - 1);
        const int np = pa.mode == 1 ? np1 : np0;
        if (np == W - 1) {
            if (TRACE) {
                if (row) {
#pragma unroll
                    for (int k = 0; k < CP_N; k++) trace[((size_t)(it - 1) * W + t) * CP_N + k] = xc[k];
                }
                if (t == 0) trace_prog[it - 1] = np;
            }
            ok = true;
            iters = it;
            prog = np;
            break;
        }
        if (vm & 1u) {   // the query is over: abandon
            aborted = true;
            break;
        }
        const bool upd = row && t > np;
#pragma unroll
        for (int k = 0; k < CP_N; k++) xc[k] = upd ? xn[k] : xc[k];
        prog = np;
        if (TRACE) {
            if (row) {
#pragma unroll
                for (int k = 0; k < CP_N; k++) trace[((size_t)(it - 1) * W + t) * CP_N + k] = xc[k];
            }
            if (t == 0) trace_prog[it - 1] = np;
        }
    }
    if (poll) pslot[8] = (int)par;
}

// Project the team's segment in place: Alg. 1 (pure.py:549-577) for modes
// 0/1, the sequential baseline (pure.py:580-615) for mode 2, then the
// clamp-and-revalidate finish (maniplan/projection.py:162-180).
// seg rows [0, W) live in shared memory; lane t owns row t.
// trace (optional, parity only): after every iteration the buffer is copied
// to trace[it-1] and the prefix to trace_prog[it-1].
// stop_flag (planner): the query's stop word, polled once per iteration
// through poll_slot (the team's 48-byte, 16-byte aligned shared-memory slot;
// no poll without it) off the critical path (cp_alg1_loop); when it is set
// the projection is abandoned (returns false with *iters_out = -1) so a team
// that lost the race leaves within two iterations instead of finishing its
// projection.
// The outcome travels back in registers (a struct return of the out-of-line
// body; cp_project below is the inline adapter): out-pointers into the
// caller's frame would pin its locals in local memory.
struct ProjRes {
    bool ok;
    int iters, prog;   // iters < 0: abandoned (the query is over)
    unsigned s1;       // stage-1 evaluations
};

__device__ __noinline__ ProjRes cp_project_body(const Team tm, float (*seg)[CP_NP], int W, const ProjArgs pa,
                                                float* trace, int* trace_prog, const int* stop_flag,
                                                int* poll_slot) {
    unsigned s1 = 0;
    const int t = (int)tm.lane;
    const bool row = t < W;
    float tau_sm = pa.tau_sm_fixed;
    if (!(tau_sm > 0.f)) {   // _resolve_taus (projection.py:137-144)
        float g = 0.f;
        if (row && t >= 1) {
            float s2 = 0.f;
#pragma unroll
            for (int k = 0; k < CP_N; k++) { float d = seg[t][k] - seg[t - 1][k]; s2 += d * d; }
            g = sqrtf(s2);
        }
        // max over the team in one REDUX: non-negative floats order as their
        // bit patterns; NaN drops out as in fmaxf (an all-NaN team gives 0,
        // and so the same 1e-6 as NaN would below)
        g = __uint_as_float(__reduce_max_sync(tm.mask, g == g ? __float_as_uint(g) : 0u));
        tau_sm = g > 0.f ? 1.5f * g : 1e-6f;
    }
    int prog = 0, iters = pa.max_iters;
    bool ok = false;
    if (pa.mode == 2) {
        // sequential: converge waypoint t before t+1 (one lane active at a time)
        int total = 0;
        ok = true;
        for (int w = 1; w < W && ok; w++) {
            int res = 0, its = 0;
            if (t == w) {
                float q[CP_N];
#pragma unroll
                for (int k = 0; k < CP_N; k++) q[k] = seg[w][k];
                res = 1;
                for (;;) {
                    bool fin = true;
#pragma unroll
                    for (int k = 0; k < CP_N; k++) fin &= cp_finite(q[k]);
                    if (!fin) { res = 0; break; }
                    float e[CP_M], J[CP_M][CP_N], st[CP_N], en2 = 0.f;
                    cp_err_jac_f(cp_conf, q, e, J);
#pragma unroll
                    for (int i = 0; i < CP_M; i++) en2 += e[i] * e[i];
                    if (sqrtf(en2) < pa.tau_task_dev) break;
                    if (its == pa.max_iters) { res = 0; break; }
                    if (!cp_damped<float, CP_M>(J, e, pa.lam, st)) { res = 0; break; }
#pragma unroll
                    for (int k = 0; k < CP_N; k++) q[k] = q[k] - pa.alpha * st[k];
                    its++;
                }
                if (res) {
                    float s2 = 0.f;
#pragma unroll
                    for (int k = 0; k < CP_N; k++) { float d = q[k] - seg[w - 1][k]; s2 += d * d; }
                    if (!(sqrtf(s2) < tau_sm * 0.99999f)) res = 0;
                }
                if (res) {
#pragma unroll
                    for (int k = 0; k < CP_N; k++) seg[w][k] = q[k];
                }
            }
            res = tm.bcast(res, w);
            its = tm.bcast(its, w);
            tm.sync();
            if (!res) { ok = false; prog = w - 1; }
            else total += its;
        }
        if (ok) { prog = W - 1; iters = total; }
    } else {
        // each lane keeps its row in registers across iterations and takes the
        // previous row from lane t-1 by shuffle (no shared-memory round trip);
        // the rows go back to seg when the loop ends
        float xc[CP_N];
#pragma unroll
        for (int k = 0; k < CP_N; k++) xc[k] = row ? seg[t][k] : 0.f;
        bool aborted = false;
        // one loop per (constrained, traced) case: the constrained planner loop
        // has no data-dependent branch besides its exits
        if (!(pa.tau_task_dev < cp_inf())) {
            if (trace) cp_alg1_loop<true, true>(tm, W, pa, tau_sm, xc, prog, iters, ok, aborted, s1, stop_flag, poll_slot, trace, trace_prog);
            else cp_alg1_loop<true, false>(tm, W, pa, tau_sm, xc, prog, iters, ok, aborted, s1, stop_flag, poll_slot, nullptr, nullptr);
        } else {
            if (trace) cp_alg1_loop<false, true>(tm, W, pa, tau_sm, xc, prog, iters, ok, aborted, s1, stop_flag, poll_slot, trace, trace_prog);
            else cp_alg1_loop<false, false>(tm, W, pa, tau_sm, xc, prog, iters, ok, aborted, s1, stop_flag, poll_slot, nullptr, nullptr);
        }
        tm.sync();
        if (row) {
#pragma unroll
            for (int k = 0; k < CP_N; k++) seg[t][k] = xc[k];
        }
        tm.sync();
        if (aborted) return ProjRes{false, -1, prog, __reduce_add_sync(tm.mask, s1)};
    }
    if (ok) {
        // clamp to limits; if anything moved, re-check both tolerances
        float q[CP_N], qc[CP_N];
        bool moved = false;
        if (row) {
#pragma unroll
            for (int k = 0; k < CP_N; k++) {
                q[k] = seg[t][k];
                // row 0 is the fixed start (an existing tree node): never clamped
                qc[k] = t == 0 ? q[k] : fminf(fmaxf(q[k], cp_lo_f(k)), cp_hi_f(k));
                moved |= !(qc[k] == q[k]);
            }
        }
        if (tm.any(moved)) {
            tm.sync();
            bool good = true;
            if (row) {
#pragma unroll
                for (int k = 0; k < CP_N; k++) seg[t][k] = qc[k];
            }
            tm.sync();
            if (row) {
                good = cp_err_norm(seg[t]) < pa.tau_task_dev;   // the clamped row, from shared memory
                if (t >= 1) {
                    float s2 = 0.f;
#pragma unroll
                    for (int k = 0; k < CP_N; k++) { float d = qc[k] - seg[t - 1][k]; s2 += d * d; }
                    good = good && sqrtf(s2) < tau_sm * 0.99999f;
                }
            }
            if (tm.any(!good)) {
                ok = false;
                iters = pa.max_iters;
                tm.sync();   // every lane's read of seg[t - 1] above precedes the restore
                if (row) {
#pragma unroll
                    for (int k = 0; k < CP_N; k++) seg[t][k] = q[k];
                }
            }
            tm.sync();
        }
    } else {
        iters = pa.max_iters;
    }
    return ProjRes{ok, iters, prog, __reduce_add_sync(tm.mask, s1)};
}

__device__ __forceinline__ bool cp_project(const Team tm, float (*seg)[CP_NP], int W, const ProjArgs pa,
                                           int* iters_out, int* prog_out, float* trace = nullptr,
                                           int* trace_prog = nullptr, unsigned long long* n_stage1 = nullptr,
                                           const int* stop_flag = nullptr, int* poll_slot = nullptr) {
    const ProjRes r = cp_project_body(tm, seg, W, pa, trace, trace_prog, stop_flag, poll_slot);
    *iters_out = r.iters;
    *prog_out = r.prog;
    if (n_stage1) *n_stage1 += r.s1;
    return r.ok;
}

// ---------------------------------------------------------------------------
// collision checking against the smem scene (pure.py:646-699)
// ---------------------------------------------------------------------------

struct ValOut {
    bool valid;
    int first_bad;         // waypoint of the first detection in (round, waypoint) order
    i64 performed;         // lockstep-equivalent count (reference semantics), exact mode
    i64 gpu_checks;        // checks this team actually evaluated
    int fk_evals;          // waypoint FK evaluations
};

// explicit shared-space 128-bit load (the staged scene is only known to the
// compiler as a generic pointer, which would otherwise become LD.E.128)
__device__ __forceinline__ float4 cp_lds4(const float4* p) {
    float4 v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

__device__ __forceinline__ bool cp_hit_box(float cx, float cy, float cz, float r2, float4 c, float4 h) {
    float dx = fmaxf(fabsf(cx - c.x) - h.x, 0.f);
    float dy = fmaxf(fabsf(cy - c.y) - h.y, 0.f);
    float dz = fmaxf(fabsf(cz - c.z) - h.z, 0.f);
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < r2;
}
__device__ __forceinline__ bool cp_hit_sph(float cx, float cy, float cz, float r, float4 s) {
    float dx = cx - s.x, dy = cy - s.y, dz = cz - s.z, rr = r + s.w;
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr;
}

// Packed CC tests (cp_f2 helpers above).  The lockstep CC pass tests robot
// spheres s and s+1 against each staged primitive together: their centres sit
// packed per axis, a primitive coordinate is the broadcast operand, and the
// squared distance is built with the same fused operations in the same order
// as the scalar tests (cp_hit_box / cp_hit_sph), so every verdict is the
// scalar one (DESIGN.md section 3 has the instruction counts).
//
// spheres (cx, cy, cz packed) vs one box (centre c, half extent h):
// cp_hit_box for both.  The clamp max(|d| - h, 0) is an FMNMX (ALU pipe) or,
// with CP_CC_CLAMP_ALU 0, u = t + |t| = 2 max(t, 0) (t = |d| - h: FP32-pipe
// adds with |.| operand modifiers) whose squared sum, exactly 4x the scalar
// one (a power-of-two scale), is compared with 4 r^2 -- the same verdict
// either way; r40 / r41 are the radii squared times CP_CC_RSCALE.
__device__ __forceinline__ void cp_hit_box2(cp_f2 cx, cp_f2 cy, cp_f2 cz, float r40, float r41, float4 c, float4 h,
                                            bool& a0, bool& a1) {
    float dx0, dx1, dy0, dy1, dz0, dz1;
    cp_upk(cp_sub2(cx, cp_pk(c.x, c.x)), dx0, dx1);
    cp_upk(cp_sub2(cy, cp_pk(c.y, c.y)), dy0, dy1);
    cp_upk(cp_sub2(cz, cp_pk(c.z, c.z)), dz0, dz1);
    const float tx0 = fabsf(dx0) - h.x, tx1 = fabsf(dx1) - h.x, ty0 = fabsf(dy0) - h.y, ty1 = fabsf(dy1) - h.y;
    const float tz0 = fabsf(dz0) - h.z, tz1 = fabsf(dz1) - h.z;
#if CP_CC_CLAMP_ALU
    auto u2 = [](float t) { return fmaxf(t, 0.f); };      // FMNMX (ALU pipe); compare with r^2
#else
    auto u2 = [](float t) { return t + fabsf(t); };        // 2 max(t, 0) on the FP32 pipe; compare with 4 r^2
#endif
    const cp_f2 ux = cp_pk(u2(tx0), u2(tx1));
    const cp_f2 uy = cp_pk(u2(ty0), u2(ty1));
    const cp_f2 uz = cp_pk(u2(tz0), u2(tz1));
    float s0, s1;
    cp_upk(cp_fma2(ux, ux, cp_fma2(uy, uy, cp_mul2(uz, uz))), s0, s1);
    a0 |= s0 < r40;
    a1 |= s1 < r41;
}

// Robot spheres s, s+1 packed per axis (one 64-bit register pair each), the
// layout cp_env_pass loads: no repacking moves in the primitive loop.
struct SPair {
    cp_f2 x, y, z;
};
// spheres (packed centres, radii r) vs one obstacle sphere o: cp_hit_sph for both
__device__ __forceinline__ void cp_hit_sph2(cp_f2 cx, cp_f2 cy, cp_f2 cz, cp_f2 r, float4 o, bool& a0, bool& a1) {
    const cp_f2 dx = cp_sub2(cx, cp_pk(o.x, o.x)), dy = cp_sub2(cy, cp_pk(o.y, o.y)),
                dz = cp_sub2(cz, cp_pk(o.z, o.z)), rr = cp_add2(r, cp_pk(o.w, o.w));
    float s0, s1, q0, q1;
    cp_upk(cp_fma2(dx, dx, cp_fma2(dy, dy, cp_mul2(dz, dz))), s0, s1);
    cp_upk(cp_mul2(rr, rr), q0, q1);
    a0 |= s0 < q0;
    a1 |= s1 < q1;
}

// The environment checks of cp_validate for one flag setting (compile-time,
// so the flag-off pass carries no votes): updates first_r (smallest round with
// a hit), rounds_done (checks per waypoint row evaluated) and stop.
template <bool FLAG>
__device__ __forceinline__ void cp_env_pass(const Team& tm, const float4* sp, const SPair* spp, bool mine,
                                            float margin, const SceneSm& sc, int E, int& first_r, i64& rounds_done,
                                            bool& stop) {
    // Robot spheres go in pairs (s, s+1) that share every staged primitive
    // load.  first_r is the smallest sphere-major round with a hit (the
    // reference's first detection, pure.py:664-698) whatever the evaluation
    // order.  With the flag on the team stops exactly when no smaller round
    // can still hit: a sphere-s hit ends the pass at once; a sphere-(s+1) hit
    // first lets sphere s finish its primitives alone (its later rounds are
    // still smaller), then ends the pass.  The votes are the paper's shared
    // collision flag, taken once per chunk.
#pragma unroll 1
    for (int s = 0; s < CP_S && !stop; s += 2) {
        const bool two = s + 1 < CP_S;
        const float4 c0 = sp[s];
        // a missing second sphere sits far from everything, including the
        // +1e18 padding primitives of the staged scene
        const float4 c1 = two ? sp[s + 1] : make_float4(-3e18f, -3e18f, -3e18f, 0.f);
        const float ra = cp_rad_tab[s] + margin, rb = (two ? cp_rad_tab[s + 1] : 0.f) + margin;
        const float r0 = ra * ra, r1 = rb * rb, r40 = CP_CC_RSCALE * r0, r41 = CP_CC_RSCALE * r1;
        const SPair pp = spp[s >> 1];
        const cp_f2 px = pp.x, py = pp.y, pz = pp.z, pr = cp_pk(ra, rb);
        const int rb0 = s * E, rb1 = (s + 1) * E;
        const int per_chunk = two ? 2 * CP_CHUNK : CP_CHUNK;
        bool only0 = false;
#pragma unroll 1
        for (int p0 = 0; p0 < sc.nb && !stop; p0 += CP_CHUNK) {
            bool a0 = false, a1 = false;
            if (!only0) {
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++)
                    cp_hit_box2(px, py, pz, r40, r41, cp_lds4(sc.box_c + p0 + j), cp_lds4(sc.box_h + p0 + j), a0, a1);
                rounds_done += per_chunk;
            } else {
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++)
                    a0 |= cp_hit_box(c0.x, c0.y, c0.z, r0, cp_lds4(sc.box_c + p0 + j), cp_lds4(sc.box_h + p0 + j));
                rounds_done += CP_CHUNK;
            }
            if (mine && a0 && rb0 + p0 < first_r) {   // rare: locate the hit
                for (int j = 0; j < CP_CHUNK; j++)
                    if (cp_hit_box(c0.x, c0.y, c0.z, r0, sc.box_c[p0 + j], sc.box_h[p0 + j])) {
                        first_r = min(first_r, rb0 + p0 + j);
                        break;
                    }
            }
            if (mine && a1 && rb1 + p0 < first_r) {
                for (int j = 0; j < CP_CHUNK; j++)
                    if (cp_hit_box(c1.x, c1.y, c1.z, r1, sc.box_c[p0 + j], sc.box_h[p0 + j])) {
                        first_r = min(first_r, rb1 + p0 + j);
                        break;
                    }
            }
            // the flag vote every CP_VOTE chunks and at the end of the boxes:
            // later votes only add checks past the first detection (first_r is
            // exact regardless), and fewer votes keep the chunk loop tight
            if (FLAG && (((p0 / CP_CHUNK) % CP_VOTE) == CP_VOTE - 1 || p0 + CP_CHUNK >= sc.nb)) {
                const int mr = (int)__reduce_min_sync(tm.mask, (unsigned)first_r);   // one team vote
                if (mr < rb1) stop = true;
                else if (mr != CP_INTMAX) only0 = true;
            }
        }
#pragma unroll 1
        for (int p0 = 0; p0 < sc.ne && !stop; p0 += CP_CHUNK) {
            bool a0 = false, a1 = false;
            if (!only0) {
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++) cp_hit_sph2(px, py, pz, pr, cp_lds4(sc.sph + p0 + j), a0, a1);
                rounds_done += per_chunk;
            } else {
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++) a0 |= cp_hit_sph(c0.x, c0.y, c0.z, ra, cp_lds4(sc.sph + p0 + j));
                rounds_done += CP_CHUNK;
            }
            if (mine && a0 && rb0 + sc.nb + p0 < first_r) {
                for (int j = 0; j < CP_CHUNK; j++)
                    if (cp_hit_sph(c0.x, c0.y, c0.z, ra, sc.sph[p0 + j])) {
                        first_r = min(first_r, rb0 + sc.nb + p0 + j);
                        break;
                    }
            }
            if (mine && a1 && rb1 + sc.nb + p0 < first_r) {
                for (int j = 0; j < CP_CHUNK; j++)
                    if (cp_hit_sph(c1.x, c1.y, c1.z, rb, sc.sph[p0 + j])) {
                        first_r = min(first_r, rb1 + sc.nb + p0 + j);
                        break;
                    }
            }
            if (FLAG && (((p0 / CP_CHUNK) % CP_VOTE) == CP_VOTE - 1 || p0 + CP_CHUNK >= sc.ne)) {
                const int mr = (int)__reduce_min_sync(tm.mask, (unsigned)first_r);   // one team vote
                if (mr < rb1) stop = true;
                else if (mr != CP_INTMAX) only0 = true;
            }
        }
        if (only0) stop = true;   // sphere s is clean: the first sphere-(s+1) hit is the first detection
    }
}

// Validate rows [t_first, W) of seg.  Lanes run in lockstep over the
// reference's check order (robot sphere major, boxes then spheres, then the
// self pairs), so a team vote after every CP_CHUNK rounds both implements the
// early-exit flag and yields the reference's first detection exactly.
// margin inflates every robot sphere (planner safety margin; 0 for parity).
// Out of line and with rolled sphere / pair loops: one compact copy of the
// check loop keeps the planner's instruction footprint inside the I-cache.
__device__ __noinline__ ValOut cp_validate(const Team tm, const float (*seg)[CP_NP], int W, int t_first,
                                           bool flag_on, float margin, const SceneSm sc) {
    const int t = (int)tm.lane;
    const bool mine = t >= t_first && t < W;
    const int E = sc.nb + sc.ne;
    float4 sp[CP_S > 0 ? CP_S : 1];   // world sphere centres of my waypoint (local memory)
    SPair spp[CP_S > 0 ? (CP_S + 1) / 2 : 1];   // the same, pair-packed for the primitive loop
    {
        float q[CP_N];
#pragma unroll
        for (int k = 0; k < CP_N; k++) q[k] = mine ? seg[t][k] : 0.f;
        float R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
        cp_fk<float>(q, R, P, AX, OR, SPH);
#pragma unroll
        for (int s = 0; s < CP_S; s++) sp[s] = make_float4(SPH[3 * s], SPH[3 * s + 1], SPH[3 * s + 2], 0.f);
        // a missing second sphere of the last pair sits far from everything,
        // including the +1e18 padding primitives of the staged scene
#pragma unroll
        for (int s = 0; s < CP_S; s += 2) {
            const bool two = s + 1 < CP_S;
            const int u = two ? 3 * s + 3 : 3 * s;   // (in range when there is no second sphere)
            spp[s >> 1] = SPair{cp_pk(SPH[3 * s], two ? SPH[u] : -3e18f), cp_pk(SPH[3 * s + 1], two ? SPH[u + 1] : -3e18f),
                                cp_pk(SPH[3 * s + 2], two ? SPH[u + 2] : -3e18f)};
        }
    }
    int first_r = CP_INTMAX;
    i64 rounds_done = 0;   // checks per waypoint row this team evaluated (team-uniform)
    bool stop = false;
    if (flag_on) cp_env_pass<true>(tm, sp, spp, mine, margin, sc, E, first_r, rounds_done, stop);
    else cp_env_pass<false>(tm, sp, spp, mine, margin, sc, E, first_r, rounds_done, stop);
    if (!stop && CP_P > 0) {
        const int rbase = CP_S * E;
#pragma unroll 1
        for (int k = 0; k < CP_P; k++) {
            const int a = cp_pair_tab[2 * k], b = cp_pair_tab[2 * k + 1];
            const float rr = cp_rad_tab[a] + cp_rad_tab[b] + 2.f * margin;
            const float4 pa = sp[a], pb = sp[b];
            float dx = pa.x - pb.x, dy = pa.y - pb.y, dz = pa.z - pb.z;
            bool hit = fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr;
            if (mine && hit && first_r == CP_INTMAX) first_r = rbase + k;
        }
        rounds_done += CP_P;
    }
    ValOut o;
    int key = first_r, idx = t;
    tm.argmin_i(key, idx);
    const i64 per = (i64)CP_S * E + CP_P;
    o.valid = key == CP_INTMAX;
    o.first_bad = o.valid ? -1 : idx;
    const int nw = W - t_first;   // waypoints checked (the planner skips row 0, an existing node)
    o.performed = (flag_on && !o.valid) ? (i64)key * nw + (idx - t_first) + 1 : per * nw;
    o.gpu_checks = rounds_done * (W - t_first);
    o.fk_evals = W - t_first;
    return o;
}

// Broad-phase validation over the clustered scene (sc.cull): the verdict of
// cp_validate / validate_waypoints (pure.py:646-699) with far fewer checks.
// Each lane bounds its waypoint's robot spheres by one box; a chunk of 8
// primitives is skipped by the whole team unless some lane's robot box
// overlaps the chunk's bound, and then only the robot spheres that reach the
// bound test the 8 primitives.  Bounds are conservative (the host rounds them
// outward with 1e-5 m of slack), so every hit cp_validate finds is found.
// The early-exit flag is a team vote after each chunk.  Counters: performed =
// sphere-primitive checks evaluated, gpu_checks = those + bound tests;
// first_bad = lowest colliding waypoint (not the reference's lockstep order).
__device__ __forceinline__ unsigned cp_team_or(const Team& tm, unsigned v) {
    return __reduce_or_sync(tm.mask, v);
}

// Robot sphere centres of the lane's waypoint: registers when the robot has
// at most CP_SREG_MAX spheres (every access below then has a compile-time
// index -- unrolled loops, the self pairs through the folded cp_pair_a/b
// switches, and a select chain for the narrow phase's warp-uniform sphere
// index), else a local array (dynamically indexed: the 36-sphere arm).
#define CP_SREG_MAX 16
#define CP_SREG (CP_S > 0 && CP_S <= CP_SREG_MAX)
#ifndef CP_NARROW_PAIRS
#define CP_NARROW_PAIRS 1   // register path: narrow phase by packed sphere pairs (else bit loop + select chain)
#endif

__device__ __noinline__ ValOut cp_validate_cull(const Team tm, const float (*seg)[CP_NP], int W, int t_first,
                                                bool flag_on, float margin, const SceneSm sc) {
    const int t = (int)tm.lane;
    const bool mine = t >= t_first && t < W;
#if CP_SREG
    float sx[CP_S], sy[CP_S], sz[CP_S], sr[CP_S];
#define CP_SPH(s) make_float4(sx[s], sy[s], sz[s], sr[s])
#else
    float4 sp[CP_S > 0 ? CP_S : 1];
#define CP_SPH(s) sp[s]
#endif
    float4 rc, rh;   // robot box of my waypoint (centre / half extent)
    {
        float q[CP_N];
#pragma unroll
        for (int k = 0; k < CP_N; k++) q[k] = mine ? seg[t][k] : 0.f;
        float R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
        cp_fk<float>(q, R, P, AX, OR, SPH);
        float lx = cp_inf(), ly = cp_inf(), lz = cp_inf(), hx = -cp_inf(), hy = -cp_inf(), hz = -cp_inf();
#pragma unroll
        for (int s = 0; s < CP_S; s++) {
            const float r = cp_rad_tab[s] + margin;
#if CP_SREG
            sx[s] = SPH[3 * s]; sy[s] = SPH[3 * s + 1]; sz[s] = SPH[3 * s + 2]; sr[s] = r;
#else
            sp[s] = make_float4(SPH[3 * s], SPH[3 * s + 1], SPH[3 * s + 2], r);
#endif
            lx = fminf(lx, SPH[3 * s] - r); hx = fmaxf(hx, SPH[3 * s] + r);
            ly = fminf(ly, SPH[3 * s + 1] - r); hy = fmaxf(hy, SPH[3 * s + 1] + r);
            lz = fminf(lz, SPH[3 * s + 2] - r); hz = fmaxf(hz, SPH[3 * s + 2] + r);
        }
        rc = make_float4(0.5f * (lx + hx), 0.5f * (ly + hy), 0.5f * (lz + hz), 0.f);
        // idle lanes get an empty box (never overlaps)
        rh = mine ? make_float4(0.5f * (hx - lx) + 1e-5f, 0.5f * (hy - ly) + 1e-5f, 0.5f * (hz - lz) + 1e-5f, 0.f)
                  : make_float4(-1e30f, -1e30f, -1e30f, 0.f);
    }
    // sphere s (warp-uniform, runtime) of the narrow phase
    auto sph_at = [&](int s) -> float4 {
#if CP_SREG
        float4 c = CP_SPH(0);
#pragma unroll
        for (int i = 1; i < CP_S; i++)
            if (s == i) c = CP_SPH(i);
        return c;
#else
        return sp[s];
#endif
    };
    // robot spheres that reach a chunk bound (bc, bh): one bit per sphere,
    // tested two spheres per packed FP32x2 step (cp_hit_box2 = cp_hit_box)
    auto bound_mask = [&](float4 bc, float4 bh, unsigned* m) {
#pragma unroll
        for (int s = 0; s + 1 < CP_S; s += 2) {
            const float4 a = CP_SPH(s), b = CP_SPH(s + 1);
            bool h0 = false, h1 = false;
            cp_hit_box2(cp_pk(a.x, b.x), cp_pk(a.y, b.y), cp_pk(a.z, b.z), CP_CC_RSCALE * (a.w * a.w),
                        CP_CC_RSCALE * (b.w * b.w), bc, bh, h0, h1);
            m[s >> 5] |= (h0 ? 1u << (s & 31) : 0u) | (h1 ? 1u << ((s + 1) & 31) : 0u);
        }
        if (CP_S & 1) {
            const float4 a = CP_SPH(CP_S - 1);
            if (cp_hit_box(a.x, a.y, a.z, a.w * a.w, bc, bh)) m[(CP_S - 1) >> 5] |= 1u << ((CP_S - 1) & 31);
        }
    };
    bool hit = false, stop = false;
    i64 narrow = 0, bound = 0;
    const float4* cl = sc.cl;
    // superchunk bounds (8 chunks each) after the chunks: a group the team's
    // robot boxes miss skips all 64 of its primitives with one test and vote
    const int nbg = (sc.nbc + 7) >> 3, neg = (sc.nec + 7) >> 3;
    const float4* gb = cl + CP_BCH * sc.nbc + CP_SCH * sc.nec;
    const float4* gs = gb + 2 * nbg;
#pragma unroll 1
    for (int g = 0; g < nbg && !stop; g++) {
    {
        const float4 gc = cp_lds4(gb + 2 * g), gh = cp_lds4(gb + 2 * g + 1);
        const bool gov = fabsf(rc.x - gc.x) <= rh.x + gh.x && fabsf(rc.y - gc.y) <= rh.y + gh.y &&
                         fabsf(rc.z - gc.z) <= rh.z + gh.z;
        if (!tm.any(gov)) continue;
    }
    const int kend = min(8 * g + 8, sc.nbc);
#pragma unroll 1
    for (int k = 8 * g; k < kend && !stop; k++) {
        const float4* ch = cl + CP_BCH * k;
        const float4 bc = cp_lds4(ch), bh = cp_lds4(ch + 1);
        const bool ov = fabsf(rc.x - bc.x) <= rh.x + bh.x && fabsf(rc.y - bc.y) <= rh.y + bh.y &&
                        fabsf(rc.z - bc.z) <= rh.z + bh.z;
        if (!tm.any(ov)) continue;
        unsigned m[(CP_S + 31) / 32 > 0 ? (CP_S + 31) / 32 : 1] = {};
        if (ov) {
            bound_mask(bc, bh, m);
            bound += CP_S;
        }
#if CP_SREG && CP_NARROW_PAIRS
        {   // sphere pairs with a reaching member test the 8 boxes packed (no
            // select chain for a runtime sphere index, no per-sphere loop)
            const unsigned um = cp_team_or(tm, m[0]);
#pragma unroll
            for (int s = 0; s < CP_S; s += 2) {
                if ((um >> s) & 3u) {
                    const float4 a = CP_SPH(s), b = CP_SPH(s + 1 < CP_S ? s + 1 : s);
                    const cp_f2 px = cp_pk(a.x, b.x), py = cp_pk(a.y, b.y), pz = cp_pk(a.z, b.z);
                    const float ra = CP_CC_RSCALE * (a.w * a.w), rb = CP_CC_RSCALE * (b.w * b.w);
                    bool h0 = false, h1 = false;
#pragma unroll
                    for (int j = 0; j < CP_CHUNK; j++)
                        cp_hit_box2(px, py, pz, ra, rb, cp_lds4(ch + 2 + j), cp_lds4(ch + 2 + CP_CHUNK + j), h0, h1);
                    const unsigned mine = (m[0] >> s) & (s + 1 < CP_S ? 3u : 1u);
                    hit |= ((mine & 1u) && h0) || ((mine & 2u) && h1);
                    narrow += CP_CHUNK * __popc(mine);
                }
            }
        }
#else
#pragma unroll
        for (int w = 0; w < (CP_S + 31) / 32; w++) {
            unsigned um = cp_team_or(tm, m[w]);
#pragma unroll 1
            while (um) {
                const int s = 32 * w + __ffs(um) - 1;
                um &= um - 1;
                const float4 c = sph_at(s);
                const float r2 = c.w * c.w;
                bool any = false;
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++)
                    any |= cp_hit_box(c.x, c.y, c.z, r2, cp_lds4(ch + 2 + j), cp_lds4(ch + 2 + CP_CHUNK + j));
                if ((m[w] >> (s & 31)) & 1u) { hit |= any; narrow += CP_CHUNK; }
            }
        }
#endif
        if (flag_on && tm.any(hit)) stop = true;   // the shared collision flag
    }
    }
    const float4* cs = cl + CP_BCH * sc.nbc;
#pragma unroll 1
    for (int g = 0; g < neg && !stop; g++) {
    {
        const float4 gc = cp_lds4(gs + 2 * g), gh = cp_lds4(gs + 2 * g + 1);
        const bool gov = fabsf(rc.x - gc.x) <= rh.x + gh.x && fabsf(rc.y - gc.y) <= rh.y + gh.y &&
                         fabsf(rc.z - gc.z) <= rh.z + gh.z;
        if (!tm.any(gov)) continue;
    }
    const int kend = min(8 * g + 8, sc.nec);
#pragma unroll 1
    for (int k = 8 * g; k < kend && !stop; k++) {
        const float4* ch = cs + CP_SCH * k;
        const float4 bc = cp_lds4(ch), bh = cp_lds4(ch + 1);
        const bool ov = fabsf(rc.x - bc.x) <= rh.x + bh.x && fabsf(rc.y - bc.y) <= rh.y + bh.y &&
                        fabsf(rc.z - bc.z) <= rh.z + bh.z;
        if (!tm.any(ov)) continue;
        unsigned m[(CP_S + 31) / 32 > 0 ? (CP_S + 31) / 32 : 1] = {};
        if (ov) {
            bound_mask(bc, bh, m);
            bound += CP_S;
        }
#if CP_SREG && CP_NARROW_PAIRS
        {
            const unsigned um = cp_team_or(tm, m[0]);
#pragma unroll
            for (int s = 0; s < CP_S; s += 2) {
                if ((um >> s) & 3u) {
                    const float4 a = CP_SPH(s), b = CP_SPH(s + 1 < CP_S ? s + 1 : s);
                    const cp_f2 px = cp_pk(a.x, b.x), py = cp_pk(a.y, b.y), pz = cp_pk(a.z, b.z), pr = cp_pk(a.w, b.w);
                    bool h0 = false, h1 = false;
#pragma unroll
                    for (int j = 0; j < CP_CHUNK; j++) cp_hit_sph2(px, py, pz, pr, cp_lds4(ch + 2 + j), h0, h1);
                    const unsigned mine = (m[0] >> s) & (s + 1 < CP_S ? 3u : 1u);
                    hit |= ((mine & 1u) && h0) || ((mine & 2u) && h1);
                    narrow += CP_CHUNK * __popc(mine);
                }
            }
        }
#else
#pragma unroll
        for (int w = 0; w < (CP_S + 31) / 32; w++) {
            unsigned um = cp_team_or(tm, m[w]);
#pragma unroll 1
            while (um) {
                const int s = 32 * w + __ffs(um) - 1;
                um &= um - 1;
                const float4 c = sph_at(s);
                bool any = false;
#pragma unroll
                for (int j = 0; j < CP_CHUNK; j++) any |= cp_hit_sph(c.x, c.y, c.z, c.w, cp_lds4(ch + 2 + j));
                if ((m[w] >> (s & 31)) & 1u) { hit |= any; narrow += CP_CHUNK; }
            }
        }
#endif
        if (flag_on && tm.any(hit)) stop = true;
    }
    }
    if (!stop && CP_P > 0) {
#if CP_SREG
#pragma unroll
        for (int k = 0; k < CP_P; k++) {   // compile-time pair indices: registers only
            const float4 pa = CP_SPH(cp_pair_a(k)), pb = CP_SPH(cp_pair_b(k));
#else
#pragma unroll 1
        for (int k = 0; k < CP_P; k++) {
            const float4 pa = sp[cp_pair_tab[2 * k]], pb = sp[cp_pair_tab[2 * k + 1]];
#endif
            const float rr = pa.w + pb.w;
            float dx = pa.x - pb.x, dy = pa.y - pb.y, dz = pa.z - pb.z;
            hit |= mine && fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr;
        }
        if (mine) narrow += CP_P;
    }
#undef CP_SPH
    ValOut o;
    int key = hit ? t : CP_INTMAX, idx = t;
    tm.argmin_i(key, idx);
    o.valid = key == CP_INTMAX;
    o.first_bad = o.valid ? -1 : key;
    i64 nsum = narrow + bound;
    // team totals (lane sums; i64 as two halves)
    unsigned lo = (unsigned)narrow, lo2 = (unsigned)nsum;
    o.performed = (i64)__reduce_add_sync(tm.mask, lo);
    o.gpu_checks = (i64)__reduce_add_sync(tm.mask, lo2);
    o.fk_evals = W - t_first;
    return o;
}

// ---------------------------------------------------------------------------
// nearest neighbour: coalesced float4 SoA scan + team argmin (planner.py:198-201)
// nodes: coordinate d of node i at nodes[d * cap + i]; never-written slots are
// NaN and drop out of the comparison.  Ties go to the lowest index.
// ---------------------------------------------------------------------------
__device__ __noinline__ int cp_nearest(const Team tm, const float* nodes, int cap, int count, const float* q) {
    float qq[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) qq[k] = q[k];
    float best = cp_inf();
    int bi = CP_INTMAX;
    const int n4 = (count + 3) >> 2;
#pragma unroll 4
    for (int i4 = (int)tm.lane; i4 < n4; i4 += CP_G) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CP_N; k++) {
            float4 v = cp_ldcg4(nodes + (size_t)k * cap + 4 * i4);
            float a = v.x - qq[k], b = v.y - qq[k], cc = v.z - qq[k], d = v.w - qq[k];
            acc.x = fmaf(a, a, acc.x); acc.y = fmaf(b, b, acc.y);
            acc.z = fmaf(cc, cc, acc.z); acc.w = fmaf(d, d, acc.w);
        }
        const int i0 = 4 * i4;
        if (acc.x < best && i0 < count) { best = acc.x; bi = i0; }
        if (acc.y < best && i0 + 1 < count) { best = acc.y; bi = i0 + 1; }
        if (acc.z < best && i0 + 2 < count) { best = acc.z; bi = i0 + 2; }
        if (acc.w < best && i0 + 3 < count) { best = acc.w; bi = i0 + 3; }
    }
    tm.argmin(best, bi);
    return bi == CP_INTMAX ? 0 : bi;
}

// The planner's nearest neighbour in one L2 round trip instead of three: the
// first chunk (nodes 4 lane .. 4 lane + 3) is loaded together with the tree's
// node counter -- slots past the end are NaN (never written, or refilled by
// the previous run's cp_reset_kernel) and drop out, and nodes appended after
// the counter was read are legitimate tree nodes -- and each lane keeps the
// coordinates of its best node, so the winner's configuration comes from a
// shuffle instead of a reload.  Writes it to out (lanes < CP_N), the node
// count to *count_out; same argmin and ties as cp_nearest.
__device__ __noinline__ int cp_nearest_ld(const Team tm, const float* nodes, int cap, const int* cnt,
                                          const float* q, float* out, int* count_out) {
    float qq[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) qq[k] = q[k];
    const int lane = (int)tm.lane;
    float4 v[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) v[k] = cp_ldcg4(nodes + (size_t)k * cap + 4 * lane);   // 4 CP_G <= 128 <= cap
    int count = lane == 0 ? cp_ldvol(cnt) : 0;
    count = min(tm.bcast(count, 0), cap);
    float best = cp_inf(), bc[CP_N];
    int bi = CP_INTMAX;
    auto take = [&](const float4* w, int i0) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CP_N; k++) {
            float a = w[k].x - qq[k], b = w[k].y - qq[k], cc = w[k].z - qq[k], d = w[k].w - qq[k];
            acc.x = fmaf(a, a, acc.x); acc.y = fmaf(b, b, acc.y);
            acc.z = fmaf(cc, cc, acc.z); acc.w = fmaf(d, d, acc.w);
        }
        const bool tx = acc.x < best;
        best = tx ? acc.x : best; bi = tx ? i0 : bi;
        const bool ty = acc.y < best;
        best = ty ? acc.y : best; bi = ty ? i0 + 1 : bi;
        const bool tz = acc.z < best;
        best = tz ? acc.z : best; bi = tz ? i0 + 2 : bi;
        const bool tw = acc.w < best;
        best = tw ? acc.w : best; bi = tw ? i0 + 3 : bi;
#pragma unroll
        for (int k = 0; k < CP_N; k++)
            bc[k] = tw ? w[k].w : (tz ? w[k].z : (ty ? w[k].y : (tx ? w[k].x : bc[k])));
    };
#pragma unroll
    for (int k = 0; k < CP_N; k++) bc[k] = 0.f;
    take(v, 4 * lane);
    const int n4 = (count + 3) >> 2;
    int i4 = lane + CP_G;
#if CP_NN_PAIRS
    // two chunks per round trip: their loads are issued together (a tree of
    // ~500 nodes is ~8 chunks per lane: 4 L2 round trips instead of 8)
    for (; i4 + CP_G < n4; i4 += 2 * CP_G) {
        float4 u[CP_N];
#pragma unroll
        for (int k = 0; k < CP_N; k++) {
            v[k] = cp_ldcg4(nodes + (size_t)k * cap + 4 * i4);
            u[k] = cp_ldcg4(nodes + (size_t)k * cap + 4 * (i4 + CP_G));
        }
        take(v, 4 * i4);
        take(u, 4 * (i4 + CP_G));
    }
#endif
    for (; i4 < n4; i4 += CP_G) {
#pragma unroll
        for (int k = 0; k < CP_N; k++) v[k] = cp_ldcg4(nodes + (size_t)k * cap + 4 * i4);
        take(v, 4 * i4);
    }
    const int my_bi = bi;
    tm.argmin(best, bi);
    const unsigned own = tm.ballot(my_bi == bi && bi != CP_INTMAX);
    const int src = own ? __ffs(own) - 1 : 0;
    float x = 0.f;
#pragma unroll
    for (int k = 0; k < CP_N; k++) {
        const float c = __shfl_sync(tm.mask, bc[k], src, CP_G);
        x = lane == k ? c : x;
    }
    tm.sync();   // every lane's reads of the previous contents of out are done
    if (lane < CP_N) out[lane] = x;
    tm.sync();
    *count_out = count;
    return bi == CP_INTMAX ? 0 : bi;
}

// ---------------------------------------------------------------------------
// Halton sampling, FP64, bit-exact with maniplan/sampling.py:32-81
// ---------------------------------------------------------------------------
// the k-th prime (k < 32) from four packed immediates: no table load (a
// cold constant-bank miss right after an L2 flush costs a DRAM round trip)
__device__ __forceinline__ int cp_prime(int k) {
    const u64 p0 = 0x13110d0b07050302ull, p1 = 0x352f2b29251f1d17ull;
    const u64 p2 = 0x59534f4947433d3bull, p3 = 0x837f716d6b676561ull;
    const u64 w = k < 8 ? p0 : (k < 16 ? p1 : (k < 24 ? p2 : p3));
    return (int)((w >> (8 * (k & 7))) & 0xffull);
}
__device__ __forceinline__ double cp_radical_inverse(i64 index, int base) {
    double f = 0.0;
    const double b = (double)base;
    double scale = __ddiv_rn(1.0, b);
    i64 i = index;
    while (i > 0) {
        f = __dadd_rn(f, __dmul_rn((double)(i % base), scale));
        scale = __ddiv_rn(scale, b);
        i /= base;
    }
    return f;
}
// The same operations without the per-digit FP64 division and 64-bit integer
// division: the scale sequence is the generated table cp_hscale (the
// reference's own values, bit for bit) and i / b is a 64-bit multiply-high by
// cp_hmagic (exact for i < 2^32).  k = joint index (base = k-th prime).
// Base 2 (k = 0): every term and partial sum is a dyadic rational with at
// most 32 significant bits, so the reference's sum is exactly the bit
// reversal of the index times 2^-32.
__device__ __forceinline__ double cp_radical_inverse_k(i64 index, int k) {
    if (index < 0 || index >= (1ll << 32)) return cp_radical_inverse(index, cp_prime(k));
    if (k == 0) return __dmul_rn((double)__brev((unsigned)index), 0x1p-32);
    const u64 M = cp_hmagic[k], b = (u64)cp_prime(k);
    const double* sc = cp_hscale[k];
    u64 i = (u64)index;
    double f = 0.0;
    for (int d = 0; i > 0; d++) {
        const u64 q = __umul64hi(i << 24, M);
        f = __dadd_rn(f, __dmul_rn((double)(unsigned)(i - q * b), sc[d]));
        i = q;
    }
    return f;
}
// pull joint k's Halton tables toward the SM (kernel prologues: after an L2
// flush their first use would otherwise wait on DRAM inside the sample)
__device__ __forceinline__ void cp_halton_prefetch(int k) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(&cp_hmagic[k]));
#pragma unroll
    for (int d = 0; d < 48; d += 16) asm volatile("prefetch.global.L1 [%0];" ::"l"(&cp_hscale[k][d]));
}
__device__ __forceinline__ double cp_halton(i64 index, int k) {
    double u = cp_radical_inverse_k(index, k);
    return __dadd_rn(cp_lo(k), __dmul_rn(__dsub_rn(cp_hi(k), cp_lo(k)), u));
}

// ---------------------------------------------------------------------------
// small team vector helpers (lanes k < CP_N own coordinate k)
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool cp_vec_equal(const Team& tm, const float* a, const float* b) {
    bool ne = (int)tm.lane < CP_N && !(a[tm.lane] == b[tm.lane]);
    return !tm.any(ne);
}
__device__ __forceinline__ float cp_vec_dist(const Team& tm, const float* a, const float* b) {
    float d = 0.f;
    if ((int)tm.lane < CP_N) { d = a[tm.lane] - b[tm.lane]; d = d * d; }
    return sqrtf(tm.sum(d));
}
// steer (planner.py:204-211)
__device__ __forceinline__ void cp_steer(const Team& tm, const float* qn, const float* qr, float step, float* out) {
    float dist = cp_vec_dist(tm, qn, qr);
    if ((int)tm.lane < CP_N) {
        int k = tm.lane;
        out[k] = dist <= step ? qr[k] : qn[k] + (step / dist) * (qr[k] - qn[k]);
    }
    tm.sync();
}
// interpolate_segment (projection.py:114-128): endpoints stored exactly
__device__ __forceinline__ void cp_interp(const Team& tm, float (*seg)[CP_NP], int W, const float* a, const float* b) {
    const int t = tm.lane;
    tm.sync();
    if (t < W) {
        float f = (float)t / (float)(W - 1);
#pragma unroll
        for (int k = 0; k < CP_N; k++) {
            float v = a[k] + f * (b[k] - a[k]);
            seg[t][k] = t == 0 ? a[k] : (t == W - 1 ? b[k] : v);
        }
    }
    tm.sync();
}
__device__ __forceinline__ void cp_copy(const Team& tm, float* dst, const float* src) {
    tm.sync();
    if ((int)tm.lane < CP_N) dst[tm.lane] = src[tm.lane];
    tm.sync();
}

// ===========================================================================
// Planner (maniplan/planner.py:361-485) -- persistent kernel
// ===========================================================================



__device__ __forceinline__ float* cp_tree(const PlanArgs& A, int q, int k) {
    return A.trees + ((size_t)(2 * q + k) * CP_N) * A.cap;
}
__device__ __forceinline__ int* cp_par(const PlanArgs& A, int q, int k) {
    return A.parents + (size_t)(2 * q + k) * A.cap;
}

// (host mirror: runtime.cpp ws_bytes = 64 + (G + 7) NP floats, rounded up to 16 B)
struct alignas(16) TeamWS {
    int poll[16];          // stop-word polls: two 16 B landing slots + the next slot's parity (cp_alg1_loop),
                           // and at [12, 16) the connect loop's slot (cp_stop_poll_issue)
    float seg[CP_G][CP_NP];
    float qr[CP_NP], qn[CP_NP], qs[CP_NP], qe[CP_NP], qc[CP_NP], qt[CP_NP], qm[CP_NP];
};

// Stop polls around waits that cover an L2 round trip: lane 0 copies the stop
// word's 16-byte sector into the team's slot asynchronously (cp.async.cg: L2,
// no register scoreboard) and reads it after the wait.  Warp P issues one
// when a connect motion starts and reads it after the motion's wait for C's
// verdict; warp C issues one before each collision check and reads it after
// the check and the append, reporting a finished query to P with its verdict.
// Without them, short projections (one or two Alg. 1 iterations: their own
// poll is read from the second iteration on) let a team run several more
// motions after the query is solved, and the host waits for the last team.
__device__ __forceinline__ void cp_stop_poll_issue(const Team& tm, TeamWS& ws, const int* stop) {
    if (tm.lane == 0)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16; cp.async.commit_group;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&ws.poll[12])), "l"((unsigned long long)stop & ~15ull) : "memory");
}
__device__ __forceinline__ bool cp_stop_poll_read(const Team& tm, TeamWS& ws, const int* stop) {
    int v = 0;
    if (tm.lane == 0) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        v = ws.poll[12 + (int)(((unsigned long long)stop & 15ull) >> 2)];
    }
    return tm.bcast(v, 0) != 0;
}

struct Stats {
    unsigned long long v[ST_NSTAT];
    __device__ Stats() {
#pragma unroll
        for (int i = 0; i < ST_NSTAT; i++) v[i] = 0ull;
    }
};

__device__ __forceinline__ bool cp_should_stop(const Team& tm, QueryState& Q, const PlanArgs& A) {
    int s = 0;
    if (tm.lane == 0) {
        s = cp_ldvol(&Q.solved) | cp_ldvol(&Q.stop);
        if (!s && A.race_flag && cp_ldvol(A.race_flag)) {   // another racer solved the query
            Q.race_stopped = 1;
            atomicExch(&Q.stop, 1);
            s = 1;
        }
        // budget_ns < 0: a zero / negative time budget, expired before the
        // first sample (the reference's TimedOut at iteration 1, planner.py:450-453)
        if (!s && A.budget_ns != 0 && (A.budget_ns < 0 || cp_clock_ns() - Q.t0_ns > (u64)A.budget_ns)) {
            atomicExch(&Q.timed_out, 1);
            atomicExch(&Q.stop, 1);
            s = 1;
        }
    }
    return tm.bcast(s, 0) != 0;
}

// validate with stats accumulation; waypoint 0 (an existing tree node) skipped
__device__ __forceinline__ bool cp_check_motion(const Team& tm, TeamWS& ws, const PlanArgs& A,
                                                const SceneSm& sc, Stats& st) {
    // every waypoint, row 0 included: the reference validates the whole
    // derived motion (planner.py:232-236), and a tree node (the endpoint of an
    // earlier P1 projection) is itself never validated -- only its derived
    // edge, whose last row the re-projection may have moved.  Lane 0 is idle
    // during CC otherwise, so the extra row costs no latency.
    ValOut v = sc.cull ? cp_validate_cull(tm, ws.seg, A.W, 0, A.flag_on, A.margin, sc)
                       : cp_validate(tm, ws.seg, A.W, 0, A.flag_on, A.margin, sc);
    st.v[ST_CCPERF] += v.performed;     // reference (lockstep) semantics, pure.py:664-698
    st.v[ST_CCPOSS] += (u64)((i64)CP_S * (sc.nb + sc.ne) + CP_P) * A.W;
    st.v[ST_GPUCHK] += v.gpu_checks;
    st.v[ST_FKCC] += v.fk_evals;
    if (!v.valid) st.v[ST_CREJ]++;
    return v.valid;
}

// derive_edge (planner.py:223-245): the motion a->b re-derivable from its endpoints
__device__ __noinline__ bool cp_derive_edge(const Team& tm, TeamWS& ws, const PlanArgs& A, const SceneSm& sc,
                               const float* a, const float* b, Stats& st, const int* stop = nullptr,
                               unsigned long long* prof = nullptr, int* cc_poll = nullptr) {
    const long long t0 = prof ? clock64() : 0;
    cp_interp(tm, ws.seg, A.W, a, b);
    int it, pr;
    bool okp = cp_project(tm, ws.seg, A.W, A.pa, &it, &pr, nullptr, nullptr, &st.v[ST_STAGE1], stop, ws.poll);
    const long long t1 = prof ? clock64() : 0;
    if (prof) { prof[0] += (unsigned long long)(t1 - t0); prof[5] += it > 0 ? it : 0; }
    if (it < 0) return false;   // abandoned: the query is over
    st.v[ST_PROJITER] += it;
    if (!okp) {
        st.v[ST_PFAIL]++;
        return false;
    }
    if (cc_poll) {   // the certifier's stop poll, read after the check and the append
        cp_stop_poll_issue(tm, ws, stop);
        *cc_poll = 1;
    }
    const bool ok = cp_check_motion(tm, ws, A, sc, st);
    if (prof) prof[1] += (unsigned long long)(clock64() - t1);
    return ok;
}

// append q to tree k of query qi with parent par; returns index or -1 (full)
__device__ __forceinline__ int cp_append(const Team& tm, const PlanArgs& A, QueryState& Q, int qi, int k,
                                         const float* q, int par) {
    int idx = 0;
    if (tm.lane == 0) idx = atomicAdd(&Q.count[k], 1);
    idx = tm.bcast(idx, 0);
    if (idx >= A.cap) {
        if (tm.lane == 0) { atomicExch(&Q.overflow, 1); atomicExch(&Q.stop, 1); }
        return -1;
    }
    // Plain stores, no ordering between them: coordinates are published by
    // being non-NaN (a reader skips a node until every coordinate is), the
    // parent by being >= 0 -- the reset kernel returns every used slot to NaN /
    // -1 after each run, and the path extraction waits for a parent it reads
    // as -1 (the store of a node it can see is in flight), so no reader can
    // take a previous run's parent and no writer pays a fence.
    float* row = cp_tree(A, qi, k) + idx;
    if (tm.lane == 0) cp_par(A, qi, k)[idx] = par;
    if ((int)tm.lane < CP_N) row[(size_t)tm.lane * A.cap] = q[tm.lane];
    tm.sync();
    return idx;
}

__device__ __forceinline__ int cp_count(const PlanArgs& A, QueryState& Q, int k) {
    return min(cp_ldvol(&Q.count[k]), A.cap);
}

__device__ __forceinline__ void cp_load_node(const Team& tm, const PlanArgs& A, int qi, int k, int idx, float* out) {
    tm.sync();
    if ((int)tm.lane < CP_N) out[tm.lane] = __ldcg(cp_tree(A, qi, k) + (size_t)tm.lane * A.cap + idx);
    tm.sync();
}

// connect (planner.py:361-409): greedy walk of tree k toward ws.qt.
// Returns the meet node index if Reached, else -1.
__device__ __noinline__ int cp_connect(const Team& tm, TeamWS& ws, const PlanArgs& A, const SceneSm& sc,
                          QueryState& Q, int qi, int k, Stats& st, int* segments_out = nullptr) {
    int segs_added = 0;
    int cnt;
    int icur = cp_nearest_ld(tm, cp_tree(A, qi, k), A.cap, &Q.count[k], ws.qt, ws.qc, &cnt);
    st.v[ST_NNODES] += cnt;
    float dist = cp_vec_dist(tm, ws.qc, ws.qt);
    if (segments_out) *segments_out = 0;
    if (dist <= A.tol) return icur;
    for (int segs = 0; segs < A.max_connect; segs++) {
        if (segments_out) *segments_out = segs_added;
        if (segs > 0 && (segs & 3) == 0 && cp_should_stop(tm, Q, A)) return -1;   // see cp_plan_query_pair
        cp_steer(tm, ws.qc, ws.qt, A.step, ws.qs);
        cp_interp(tm, ws.seg, A.W, ws.qc, ws.qs);
        int it, pr;
        bool okp = cp_project(tm, ws.seg, A.W, A.pa, &it, &pr, nullptr, nullptr, &st.v[ST_STAGE1], &Q.stop, ws.poll);
        if (it < 0) return -1;   // abandoned: the query is over
        st.v[ST_PROJITER] += it;
        if (!okp) { st.v[ST_PFAIL]++; return -1; }
        cp_copy(tm, ws.qe, ws.seg[A.W - 1]);
        if (cp_vec_equal(tm, ws.qe, ws.qs)) {
            if (!cp_check_motion(tm, ws, A, sc, st)) return -1;
        } else if (!cp_derive_edge(tm, ws, A, sc, ws.qc, ws.qe, st, &Q.stop)) {
            return -1;
        }
        float nd = cp_vec_dist(tm, ws.qe, ws.qt);
        if (!(nd < dist)) return -1;
        int idx = cp_append(tm, A, Q, qi, k, ws.qe, icur);
        if (idx < 0) return -1;
        icur = idx;
        segs_added++;
        if (segments_out) *segments_out = segs_added;
        cp_copy(tm, ws.qc, ws.qe);
        dist = nd;
        if (dist <= A.tol) return icur;
    }
    return -1;
}

// _attempt_extend + commit (planner.py:265-325) for the sample in ws.qr against
// tree a: the new node's index, or -1 degenerate, -2 projection, -3 collision,
// -4 tree full.  ws.qe holds the new node on success.
__device__ __noinline__ int cp_extend_once(const Team& tm, TeamWS& ws, const PlanArgs& A, const SceneSm& sc,
                                           QueryState& Q, int qi, int a, Stats& st) {
    const int W = A.W;
    int cnt_a;
    const int inear = cp_nearest_ld(tm, cp_tree(A, qi, a), A.cap, &Q.count[a], ws.qr, ws.qn, &cnt_a);
    st.v[ST_NNODES] += cnt_a;
    cp_steer(tm, ws.qn, ws.qr, A.step, ws.qs);
    if (cp_vec_equal(tm, ws.qs, ws.qn)) return -1;
    cp_interp(tm, ws.seg, W, ws.qn, ws.qs);
    int pit, ppr;
    bool okp = cp_project(tm, ws.seg, W, A.pa, &pit, &ppr, nullptr, nullptr, &st.v[ST_STAGE1], &Q.stop, ws.poll);
    if (pit < 0) return -1;   // abandoned: the query is over
    st.v[ST_PROJITER] += pit;
    if (!okp) { st.v[ST_PFAIL]++; return -2; }
    cp_copy(tm, ws.qe, ws.seg[W - 1]);
    if (cp_vec_equal(tm, ws.qe, ws.qn)) return -1;
    if (cp_vec_equal(tm, ws.qe, ws.qs)) {
        if (!cp_check_motion(tm, ws, A, sc, st)) return -3;
    } else {
        const unsigned long long pf0 = st.v[ST_PFAIL];
        if (!cp_derive_edge(tm, ws, A, sc, ws.qn, ws.qe, st, &Q.stop)) return st.v[ST_PFAIL] != pf0 ? -2 : -3;
    }
    const int node = cp_append(tm, A, Q, qi, a, ws.qe, inear);
    return node < 0 ? -4 : node;
}

struct PairBox;
__device__ __noinline__ void cp_extract_path(const Team tm, const PlanArgs& A, int qi, int meet0, int meet1,
                                             float (*stage)[CP_NP], const PairBox* bx);   // below
__device__ __noinline__ void cp_extract_query(const Team tm, const PlanArgs& A, int qi);   // below

// add a team's counters to the query's (lane 0, the non-zero ones) and clear them
__device__ __forceinline__ void cp_flush_stats(const Team& tm, QueryState& Q, Stats& st) {
    if (tm.lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_NSTAT; i++)
            if (st.v[i]) atomicAdd(&Q.stats[i], st.v[i]);
    }
#pragma unroll
    for (int i = 0; i < ST_NSTAT; i++) st.v[i] = 0ull;
}

// ===========================================================================
// Pair mode (single queries): a team is two warps.  Warp P draws samples and
// runs the P1 projections of the extension and of the greedy connect; warp C
// certifies each motion P produced -- derive_edge's re-projection when the
// endpoint moved, the collision check, the append -- one motion behind P, so
// the certification of motion k overlaps P1 of motion k+1 (planner.py:265-306
// and :361-409 evaluated in the same order; P posts motion k+1 only after C
// accepted motion k, whose node is its parent).
// ===========================================================================
// The pair's mailbox (shared memory, in the unused half-team slot of P's
// warp): two mbarriers -- `full` (P's 16 lanes arrive after writing a job, C
// waits), `done` (C's 16 lanes arrive after finishing it, P waits) -- give the
// hand-offs release / acquire ordering without a CTA barrier.
// C's ancestor-chain cache (per tree): entries pw_anc[t][h .. h + len) are the
// node C appended last in tree t and its ancestors, root last when pw_root;
// sized to what the TeamWS slot holds beside the mailbox (48 for arm7)
#define CP_PW_FIT (((64 + (CP_G + 7) * CP_NP * 4) - (124 + 8 * CP_NP)) / 8)
#define CP_PW (CP_PW_FIT < 2 ? 2 : (CP_PW_FIT < 48 ? CP_PW_FIT : 48))
#define CP_PW_SLACK (CP_PW / 4)    // room to prepend connect nodes
struct PairBox {
    unsigned long long full, done;   // mbarriers
    int result;                      // new node index, or -2 projection, -3 collision, -4 full
    int over;                        // the query was over by the end of the job (stop word set)
    int qi, tree, parent, derive, exit;
    int p_ndone, p_pend;             // P's bookkeeping: done phases consumed, a result outstanding
    float from[CP_NP], to[CP_NP];
    int pw_h[2], pw_len[2], pw_root[2];
    int pw_anc[2][CP_PW];
#ifdef CP_PROFILE
    unsigned long long cprof[6];     // warp C clock64 phases: P2, CC, append, jobs, idle, P2 iterations
#endif
};
static_assert(sizeof(PairBox) <= sizeof(TeamWS), "the pair mailbox must fit a team workspace slot");
static_assert(CP_PW <= 4 * CP_G, "a cached chain fits the extraction's register slots");
__device__ __forceinline__ PairBox* cp_pair_box(TeamWS* slot) {
    return reinterpret_cast<PairBox*>((reinterpret_cast<unsigned long long>(slot) + 7ull) & ~7ull);
}
__device__ __forceinline__ unsigned cp_smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_mb_init(unsigned long long* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cp_smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void cp_mb_arrive(unsigned long long* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(cp_smem_addr(b)) : "memory");
}
__device__ __forceinline__ void cp_mb_wait(unsigned long long* b, int parity) {
    unsigned ok = 0;
    while (!ok) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(cp_smem_addr(b)), "r"(parity)
                     : "memory");
    }
}

// P: consume the outstanding job's completion, if any
__device__ __forceinline__ void cp_pair_wait_idle(const Team& tm, PairBox& bx) {
    tm.sync();
    if (bx.p_pend) {
        cp_mb_wait(&bx.done, bx.p_ndone & 1);
        tm.sync();
        if (tm.lane == 0) { bx.p_ndone = bx.p_ndone + 1; bx.p_pend = 0; }
    }
    tm.sync();
}

// post a certification job; from / to are team vectors (lanes < CP_N)
__device__ __forceinline__ void cp_pair_post(const Team& tm, PairBox& bx, TeamWS& wsc, int qi, int tree,
                                             int parent, bool derive, const float* from, const float* to,
                                             const float (*seg)[CP_NP], int W, int exit_job = 0) {
    cp_pair_wait_idle(tm, bx);
    if ((int)tm.lane < CP_N) { bx.from[tm.lane] = from[tm.lane]; bx.to[tm.lane] = to[tm.lane]; }
    if (!exit_job && !derive && (int)tm.lane < W)   // the P1 motion itself is the canonical edge
#pragma unroll
        for (int k = 0; k < CP_N; k++) wsc.seg[tm.lane][k] = seg[tm.lane][k];
    if (tm.lane == 0) {
        bx.qi = qi; bx.tree = tree; bx.parent = parent; bx.derive = derive ? 1 : 0; bx.exit = exit_job;
        bx.p_pend = 1;
    }
    tm.sync();
    cp_mb_arrive(&bx.full);   // every lane: release of its own writes
}

// C's verdict on the outstanding job; over |= the query was over by its end
__device__ __forceinline__ int cp_pair_result(const Team& tm, PairBox& bx, bool& over) {
    cp_pair_wait_idle(tm, bx);
    over |= tm.bcast(bx.over, 0) != 0;
    return tm.bcast(bx.result, 0);
}

__device__ int cp_check_config_d(const SetupArgs& S, const double* q, int lane, int nl, unsigned mask);   // below

// The single query's FP64 endpoint checks (planner.py:416-427), on the
// certifier warps of the first two teams before their first job (P's first
// projection takes far longer): team 0 checks the start, team 1 the goal
// (team 0 both if it is alone).  A bad endpoint stops the query at once; the
// second check to finish combines the codes as cp_check_kernel does, writes
// setup_code to the results and then the check's completion word.
__device__ __noinline__ void cp_pair_endpoint_checks(const Team& tm, const PlanArgs& A, int gteam, int n_teams) {
    const SetupArgs& S = A.chk;
    QueryState& Q = A.qs[0];
    for (int w = gteam; w < 2; w += n_teams) {
        const double* q = w == 0 ? S.starts : S.goals;
        const int code = cp_check_config_d(S, q, (int)tm.lane, CP_G, tm.mask);
        if (tm.lane == 0) {
            Q.chk_code[w] = code;
            if (code) atomicExch(&Q.stop, 1);
            __threadfence();
            if (atomicAdd(&Q.chk_cnt, 1) == 1) {   // both verdicts are in
                const int c0 = cp_ldvol(&Q.chk_code[0]), c1 = cp_ldvol(&Q.chk_code[1]);
                const int c = c0 ? c0 : (c1 ? 3 + c1 : 0);
                QueryOut& O = A.out[0];
                O.setup_code = c;
                if (c) Q.setup_code = c;
                __threadfence_system();
                *(volatile unsigned*)&O.chk_seq = (unsigned)A.seeds[1];   // the call's sequence number
            }
        }
        tm.sync();
    }
}

// warp C: certify jobs until P posts the exit job
__device__ void cp_pair_certifier(const Team& tm, TeamWS& ws, PairBox& bx, const PlanArgs& A, const SceneSm& sc) {
#ifdef CP_PROFILE
    unsigned long long cpf[6] = {};
#define CP_CPROF cpf
#else
#define CP_CPROF nullptr
#endif
    for (int nfull = 0;; nfull++) {
#ifdef CP_PROFILE
        const long long t_idle = clock64();
#endif
        cp_mb_wait(&bx.full, nfull & 1);
        tm.sync();
#ifdef CP_PROFILE
        cpf[4] += (unsigned long long)(clock64() - t_idle);
        cpf[3]++;
#endif
        if (bx.exit) break;
        const int qi = bx.qi, tree = bx.tree;
        QueryState& Q = A.qs[qi];
#ifdef CP_TIMELINE
        const u64 job_t0 = cp_clock_ns();
#endif
        Stats st;
        int res;
        bool ok;
        int polled = 0;
        int walk_tree = -1;
        if (bx.derive) {
            if ((int)tm.lane < CP_N) { ws.qr[tm.lane] = bx.from[tm.lane]; ws.qn[tm.lane] = bx.to[tm.lane]; }
            tm.sync();
            const unsigned long long pf0 = st.v[ST_PFAIL];
            ok = cp_derive_edge(tm, ws, A, sc, ws.qr, ws.qn, st, &Q.stop, CP_CPROF, &polled);
            res = ok ? 0 : (st.v[ST_PFAIL] != pf0 ? -2 : -3);
        } else {
            cp_stop_poll_issue(tm, ws, &Q.stop);
            polled = 1;
#ifdef CP_PROFILE
            const long long t_cc = clock64();
#endif
            ok = cp_check_motion(tm, ws, A, sc, st);
#ifdef CP_PROFILE
            cpf[1] += (unsigned long long)(clock64() - t_cc);
#endif
            res = ok ? 0 : -3;
        }
        if (ok) {
#ifdef CP_PROFILE
            const long long t_ap = clock64();
#endif
            if ((int)tm.lane < CP_N) ws.qe[tm.lane] = bx.to[tm.lane];
            tm.sync();
            const int node = cp_append(tm, A, Q, qi, tree, ws.qe, bx.parent);
            res = node < 0 ? -4 : node;
#ifdef CP_PROFILE
            cpf[2] += (unsigned long long)(clock64() - t_ap);
#endif
        }
#ifdef CP_PROFILE
        if (tm.lane == 0)
            for (int i = 0; i < 6; i++) bx.cprof[i] = cpf[i];
#endif
        const int over = polled && cp_stop_poll_read(tm, ws, &Q.stop);
        if (tm.lane == 0) {
#pragma unroll
            for (int i = 0; i < ST_NSTAT; i++)
                if (st.v[i]) atomicAdd(&Q.stats[i], st.v[i]);
            bx.result = res;
            bx.over = over;
            if (res >= 0) {   // the ancestor cache of tree `tree` now starts at the new node
                const int t = tree, par = bx.parent;
                if (bx.pw_len[t] > 0 && bx.pw_anc[t][bx.pw_h[t]] == par && bx.pw_h[t] > 0) {
                    const int h = bx.pw_h[t] - 1;   // a connect chain: prepend
                    bx.pw_anc[t][h] = res;
                    bx.pw_h[t] = h;
                    bx.pw_len[t] = bx.pw_len[t] + 1;
                } else {                           // a new chain: the node and its parent, ancestors below
                    bx.pw_h[t] = CP_PW_SLACK;
                    bx.pw_anc[t][CP_PW_SLACK] = res;
                    bx.pw_anc[t][CP_PW_SLACK + 1] = par;
                    bx.pw_root[t] = 0;
                    bx.pw_len[t] = 2;
                    walk_tree = t;
                }
            }
#ifdef CP_TIMELINE
            // the longest job running across the solve: (ns after the solve) & ~15 | kind
            // (1 derive ok, 2 derive failed, 3 check ok, 4 check failed)
            const u64 ts = cp_ldvol64(&Q.t_end_ns), now = cp_clock_ns();
            if (ts != 0 && job_t0 <= ts && now > ts)
                atomicMax(&Q.pad1_[0], (int)((((now - ts) >> 4) << 4) | (u64)((bx.derive ? 1 : 3) + (ok ? 0 : 1))));
#endif
        }
        walk_tree = tm.bcast(walk_tree, 0);
        tm.sync();
        cp_mb_arrive(&bx.done);   // every lane: release
        // Idle until the next job: walk the new chain's ancestors (dependent L2
        // loads) into the cache, so the team that solves the query finds its
        // path's parent chains in shared memory instead of walking them.  A
        // posted job ends the walk (non-blocking mbarrier test between steps).
        if (walk_tree >= 0 && tm.lane == 0) {
            const int t = walk_tree;
            const int* pp = cp_par(A, qi, t);
            int h = bx.pw_h[t], len = bx.pw_len[t], cur = bx.pw_anc[t][h + len - 1];
            while (h + len < CP_PW) {
                unsigned posted;
                asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; "
                             "selp.u32 %0, 1, 0, p; }"
                             : "=r"(posted) : "r"(cp_smem_addr(&bx.full)), "r"((nfull + 1) & 1) : "memory");
                if (posted) break;
                int q = cp_ldvol(pp + cur);
                if (q < 0) break;   // not landed yet: leave it to the extraction's walk
                if (q == cur) {
                    *(volatile int*)&bx.pw_root[t] = 1;
                    break;
                }
                bx.pw_anc[t][h + len] = q;
                __threadfence_block();
                *(volatile int*)&bx.pw_len[t] = ++len;
                cur = q;
            }
        }
        walk_tree = -1;
        tm.sync();
    }
}

// Developer profile of the winning team's critical path (CPRRTC_DEFINES=
// CP_PROFILE, tools/pair_profile.py): warp P's clock64 time by phase, written
// to the query's result stats by the winner in place of the counters.
#ifdef CP_PROFILE
enum { PF_LAUNCH_NS = 0, PF_TOTAL, PF_PROJ, PF_PITER, PF_WAIT, PF_NN, PF_SAMPLE, PF_STOP, PF_NSAMP, PF_NPROJ,
       PF_WINIT, PF_JUNC };
#define CP_PF_T0(v) const long long v = clock64()
#define CP_PF_ADD(i, t0) (pf[i] += (u64)(clock64() - (t0)))
#define CP_PF_INC(i, n) (pf[i] += (u64)(n))
#else
#define CP_PF_T0(v)
#define CP_PF_ADD(i, t0)
#define CP_PF_INC(i, n)
#endif

// warp P: the sampling / projection side of cp_plan_query
//
// first_it > 0 (single-query launches): the team's first sample index, handed
// out statically (team k draws k + 1; the shared counter then continues
// above n_teams), and no stop poll before it -- a team's first extension
// starts without an L2 round trip.
// junction (planner.py:466-481): the edge between q_new (tree a) and the meet
// node of tree b, derived start side -> goal side
__device__ __forceinline__ bool cp_junction(const Team& tm, TeamWS& ws, const PlanArgs& A, const SceneSm& sc, int a,
                                            const float* q_new, const float* q_meet, Stats& st, const int* stop) {
    const float* js = a == 0 ? q_new : q_meet;
    const float* jg = a == 0 ? q_meet : q_new;
    if (cp_vec_equal(tm, js, jg)) return true;
    cp_copy(tm, ws.qr, js);
    cp_copy(tm, ws.qn, jg);
    return cp_derive_edge(tm, ws, A, sc, ws.qr, ws.qn, st, stop);
}

__device__ void cp_plan_query_pair(const Team& tm, TeamWS& ws, TeamWS& wsc, PairBox& bx, const PlanArgs& A,
                                   const SceneSm& sc, int qi, int first_it, int n_teams) {
    QueryState& Q = A.qs[qi];
    Stats st;
    const int W = A.W;
#ifdef CP_PROFILE
    u64 pf[ST_NSTAT] = {};
    pf[PF_LAUNCH_NS] = cp_clock_ns() - Q.t0_ns;
    const long long pf_entry = clock64();
#endif
#ifdef CP_TIMELINE
    int why = 5;
    u64 tl_t[8] = {};
    int tl_id[8] = {}, tl_n = 0;
#define CP_TL(id) do { if (tm.lane == 0) { tl_t[tl_n & 7] = cp_clock_ns(); tl_id[tl_n & 7] = (id); } tl_n++; } while (0)
#define CP_WHY(k) (why = (k))
#else
#define CP_WHY(k) ((void)0)
#define CP_TL(id) ((void)0)
#endif
    for (int round = 0;; round++) {
        // counters go to the query every round: a solved query's result
        // carries the work finished by the time it was solved (the solving
        // team finalises it at once, without waiting for the others to leave)
        if (round > 0) cp_flush_stats(tm, Q, st);
        CP_PF_T0(t_stop); CP_TL(1);
        if (!(round == 0 && first_it > 0 && A.budget_ns >= 0) && cp_should_stop(tm, Q, A)) { CP_WHY(0); break; }
        CP_PF_ADD(PF_STOP, t_stop);
        CP_PF_T0(t_samp); CP_TL(2);
        int it = first_it;
        if (round > 0 || first_it <= 0) {
            if (tm.lane == 0) it = atomicAdd(&Q.next_sample, 1) + 1 + (first_it > 0 ? n_teams : 0);
            it = tm.bcast(it, 0);
        }
        if (it > A.max_iterations) {
            if (tm.lane == 0) atomicExch(&Q.exhausted, 1);
            break;
        }
        st.v[ST_ITER]++;
        st.v[ST_ATT]++;
        const int a = (it - 1) & 1, b = a ^ 1;
        // (round 0 of a single query: drawn in the kernel prologue)
        if ((round > 0 || first_it <= 0) && (int)tm.lane < CP_N)
            ws.qr[tm.lane] = (float)cp_halton((i64)it + Q.seed_offset, tm.lane);
        tm.sync();
        CP_PF_ADD(PF_SAMPLE, t_samp);
        CP_PF_INC(PF_NSAMP, 1);
        CP_PF_T0(t_nn); CP_TL(3);
        // extension P1 (planner.py:265-281)
        int cnt_a;
        int inear;
#if CP_ROOT_FIRST
        if (round == 0 && first_it > 0) {
            // a single query's first extension: every team starts at once and
            // no motion has been appended yet, so tree a is its root (node 0)
            // -- the root's stored coordinates without the L2 round trip
            // (nodes another team appends meanwhile are as if drawn later)
            if ((int)tm.lane < CP_N)
                ws.qn[tm.lane] = (float)(a == 0 ? A.chk.starts : A.chk.goals)[tm.lane];
            tm.sync();
            inear = 0;
            cnt_a = 1;
        } else
#endif
            inear = cp_nearest_ld(tm, cp_tree(A, qi, a), A.cap, &Q.count[a], ws.qr, ws.qn, &cnt_a);
        st.v[ST_NNODES] += cnt_a;
        cp_steer(tm, ws.qn, ws.qr, A.step, ws.qs);
        if (cp_vec_equal(tm, ws.qs, ws.qn)) continue;
        cp_interp(tm, ws.seg, W, ws.qn, ws.qs);
        CP_PF_ADD(PF_NN, t_nn);
        int pit, ppr;
        CP_PF_T0(t_p1); CP_TL(4);
        bool okp = cp_project(tm, ws.seg, W, A.pa, &pit, &ppr, nullptr, nullptr, &st.v[ST_STAGE1], &Q.stop, ws.poll);
        CP_PF_ADD(PF_PROJ, t_p1);
        CP_PF_INC(PF_NPROJ, 1);
        CP_PF_INC(PF_PITER, pit > 0 ? pit : 0);
        if (pit < 0) { CP_WHY(1); break; }
        st.v[ST_PROJITER] += pit;
        if (!okp) { st.v[ST_PFAIL]++; continue; }
        cp_copy(tm, ws.qe, ws.seg[W - 1]);
        if (cp_vec_equal(tm, ws.qe, ws.qn)) continue;
        CP_PF_T0(t_post); CP_TL(5);
        cp_pair_post(tm, bx, wsc, qi, a, inear, !cp_vec_equal(tm, ws.qe, ws.qs), ws.qn, ws.qe, ws.seg, W);
        CP_PF_ADD(PF_WAIT, t_post);
        CP_PF_T0(t_nn2); CP_TL(6);
        // greedy connect of tree b toward q_new while C certifies the extension
        cp_copy(tm, ws.qt, ws.qe);
        int cnt_b;
        int icur;
#if CP_ROOT_FIRST_CONNECT
        if (round == 0 && first_it > 0) {   // as for the extension: tree b's root, no L2 round trip
            if ((int)tm.lane < CP_N)
                ws.qc[tm.lane] = (float)(b == 0 ? A.chk.starts : A.chk.goals)[tm.lane];
            tm.sync();
            icur = 0;
            cnt_b = 1;
        } else
#endif
            icur = cp_nearest_ld(tm, cp_tree(A, qi, b), A.cap, &Q.count[b], ws.qt, ws.qc, &cnt_b);
        st.v[ST_NNODES] += cnt_b;
        float dist = cp_vec_dist(tm, ws.qc, ws.qt);
        CP_PF_ADD(PF_NN, t_nn2);
        int node = -1, meet = -1;
        bool pending_ext = true, stop = false, full = false;
        int prev = -1;          // node of the last accepted connect motion
        bool pending_con = false;
        bool over = false;      // C saw the stop word set (after its last check)
        // Speculative junction: the meet node's coordinates are known before C
        // accepts the motion that creates it (C appends exactly the posted
        // endpoint; an existing node's come from the NN), so P derives the
        // junction edge while C certifies, instead of after C's verdict.  Its
        // verdict counts only if C accepts (the reference's order of effects
        // on the trees is unchanged).  -1: not run.
        int spec = -1;
        if (dist <= A.tol) {
#if CP_SPEC_JUNC
            spec = cp_junction(tm, ws, A, sc, a, ws.qt, ws.qc, st, &Q.stop) ? 1 : 0;
#endif
            node = cp_pair_result(tm, bx, over);
            pending_ext = false;
            if (node == -4) full = true;
            if (node >= 0) meet = icur;
            if (over) { CP_WHY(7); stop = true; }
        } else {
            for (int segs = 0; segs < A.max_connect; segs++) {
                // the full stop / time-budget poll every 4th motion: a solved query
                // already stops the projections (they poll the stop word) and the
                // budget is checked at every sample (r1 A/B: -2.5 % median)
                if (segs > 0 && (segs & 3) == 0 && cp_should_stop(tm, Q, A)) { CP_WHY(2); stop = true; break; }
                cp_stop_poll_issue(tm, ws, &Q.stop);
                CP_PF_T0(t_si); CP_TL(7);
                cp_steer(tm, ws.qc, ws.qt, A.step, ws.qs);
                cp_interp(tm, ws.seg, W, ws.qc, ws.qs);
                CP_PF_ADD(PF_NN, t_si);
                int it2, pr2;
                CP_PF_T0(t_p2); CP_TL(8);
                const bool ok1 = cp_project(tm, ws.seg, W, A.pa, &it2, &pr2, nullptr, nullptr, &st.v[ST_STAGE1],
                                            &Q.stop, ws.poll);
                CP_PF_ADD(PF_PROJ, t_p2);
                CP_PF_INC(PF_NPROJ, 1);
                CP_PF_INC(PF_PITER, it2 > 0 ? it2 : 0);
                if (it2 >= 0) st.v[ST_PROJITER] += it2;
                CP_PF_T0(t_w); CP_TL(9);
                // abandoned (the query is over): leave without C's verdict on the previous motion
                if (it2 < 0) { CP_WHY(3); stop = true; break; }
                // the previous motion must be accepted before this one builds on it
                if (pending_ext) {
                    node = cp_pair_result(tm, bx, over);
                    pending_ext = false;
                    if (node < 0) { full = node == -4; break; }
                } else if (pending_con) {
                    prev = cp_pair_result(tm, bx, over);
                    pending_con = false;
                    if (prev < 0) { full = prev == -4; break; }
                    icur = prev;
                }
                CP_PF_ADD(PF_WAIT, t_w);
                if (over || cp_stop_poll_read(tm, ws, &Q.stop)) { CP_WHY(7); stop = true; break; }
                if (!ok1) { st.v[ST_PFAIL]++; break; }
                cp_copy(tm, ws.qe, ws.seg[W - 1]);
                const float nd = cp_vec_dist(tm, ws.qe, ws.qt);
                if (!(nd < dist)) break;
                CP_PF_T0(t_w2); CP_TL(10);
                cp_pair_post(tm, bx, wsc, qi, b, icur, !cp_vec_equal(tm, ws.qe, ws.qs), ws.qc, ws.qe, ws.seg, W);
                pending_con = true;
                cp_copy(tm, ws.qc, ws.qe);
                dist = nd;
                CP_PF_ADD(PF_WAIT, t_w2);
                if (dist <= A.tol) {
#if CP_SPEC_JUNC
                    spec = cp_junction(tm, ws, A, sc, a, ws.qt, ws.qc, st, &Q.stop) ? 1 : 0;
#endif
                    CP_PF_T0(t_w3); CP_TL(11);
                    const int r = cp_pair_result(tm, bx, over);
                    CP_PF_ADD(PF_WAIT, t_w3);
                    pending_con = false;
                    if (r >= 0) meet = r;
                    else full = r == -4;
                    if (over) { CP_WHY(7); stop = true; }   // someone else won
                    break;
                }
            }
            CP_TL(13);
            // drain: motions still being certified are kept (the reference
            // appends every accepted motion of a trapped connect too) -- unless
            // the query is over: then the team leaves at once and C finishes
            // its job on its own (its append, if any, stays inside the slots
            // the reset refills: cp_reset_kernel covers the final count)
            if (!stop) {
                if (pending_ext) { node = cp_pair_result(tm, bx, over); pending_ext = false; if (node == -4) full = true; }
                if (pending_con) { const int r = cp_pair_result(tm, bx, over); if (r == -4) full = true; }
            }
        }
        if (node >= 0) st.v[ST_ADDED]++;
        if (full) {
            if (tm.lane == 0) { atomicExch(&Q.overflow, 1); atomicExch(&Q.stop, 1); }
            break;
        }
        if (stop) break;
        if (node < 0 || meet < 0) continue;
        CP_PF_T0(t_j); CP_TL(12);
        // junction (planner.py:466-481): q_new (tree a) against the meet node (tree b)
        bool ok;
        if (spec >= 0) {
            ok = spec != 0;
        } else {
            cp_load_node(tm, A, qi, b, meet, ws.qm);
            ok = cp_junction(tm, ws, A, sc, a, ws.qt, ws.qm, st, &Q.stop);
        }
        CP_PF_ADD(PF_JUNC, t_j);
        if (ok) {
            int won = 0;
#ifdef CP_PROFILE
            pf[PF_TOTAL] = (u64)(clock64() - pf_entry);
            pf[PF_WINIT] = (u64)it;
#endif
            if (tm.lane == 0 && atomicCAS(&Q.solved, 0, 1) == 0) {
#ifdef CP_PROFILE
#if CP_PROFILE == 2
                // warp C's phases (as of its last finished job) in place of P's NN / sample / stop slots
                pf[5] = bx.cprof[0]; pf[6] = bx.cprof[1]; pf[8] = bx.cprof[2]; pf[9] = bx.cprof[3];
                pf[10] = bx.cprof[4]; pf[11] = bx.cprof[5];
#endif
#pragma unroll
                for (int i = 0; i < ST_NSTAT; i++) A.out[qi].stats[i] = pf[i];
#endif
                Q.meet[a] = node;
                Q.meet[b] = meet;
                Q.t_end_ns = cp_clock_ns();
#ifdef CP_TIMELINE
                Q.pad1_[4] = (int)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
#endif
                // no fence: the stop word is only a signal to leave (the
                // finalizer reads meet / t_end after the active-count handshake)
                atomicExch(&Q.stop, 1);
                for (int r = 0; r < A.n_race; r++) *(volatile int*)A.race_peers[r] = 1;
                if (A.n_race) __threadfence_system();
                won = 1;
            }
            if (tm.bcast(won, 0)) {   // while the other teams leave
                CP_WHY(6);
                cp_extract_path(tm, A, qi, a == 0 ? node : meet, a == 0 ? meet : node, ws.seg, &bx);
                cp_flush_stats(tm, Q, st);
                __threadfence();
                cp_extract_query(tm, A, qi);   // the result is complete: counters, node counts, completion word
            }
            else CP_WHY(4);
            break;
        }
    }
    if (tm.lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_NSTAT; i++)
            if (st.v[i]) atomicAdd(&Q.stats[i], st.v[i]);
#ifdef CP_TIMELINE
        const u64 now = cp_clock_ns();
        atomicMax(&Q.pad1_[6 + why], (int)(now - Q.t0_ns));
        const u64 ts = cp_ldvol64(&Q.t_end_ns);
        if (why != 6 && ts != 0 && now > ts) {   // the phase this team was in when the query was solved
            int ph = 15;
            for (int j = tl_n - 1; j >= 0 && j >= tl_n - 8; j--)
                if (tl_t[j & 7] <= ts) { ph = tl_id[j & 7]; break; }
            atomicMax(&Q.pad1_[2], (int)((((now - ts) >> 4) << 4) | (u64)ph));
        }
#endif
    }
#undef CP_WHY
#undef CP_TL
}

// One team works on query qi until it is solved / stopped / out of samples.
// first_it / n_teams: as for cp_plan_query_pair.
__device__ void cp_plan_query(const Team& tm, TeamWS& ws, const PlanArgs& A, const SceneSm& sc, int qi,
                              int first_it, int n_teams) {
    QueryState& Q = A.qs[qi];
    Stats st;
    const int W = A.W;
    for (int round = 0;; round++) {
        if (!(round == 0 && first_it > 0 && A.budget_ns >= 0) && cp_should_stop(tm, Q, A)) break;
        int it = first_it;
        if (round > 0 || first_it <= 0) {
            if (tm.lane == 0) it = atomicAdd(&Q.next_sample, 1) + 1 + (first_it > 0 ? n_teams : 0);
            it = tm.bcast(it, 0);
        }
        if (it > A.max_iterations) {
            // out of samples: no new extensions, but extensions already in
            // flight (other teams) finish their connect
            if (tm.lane == 0) atomicExch(&Q.exhausted, 1);
            break;
        }
        st.v[ST_ITER]++;
        st.v[ST_ATT]++;
        const int a = (it - 1) & 1, b = a ^ 1;   // start tree extends on odd iterations
        // sample (sampling.py:65-81) -- FP64 Halton, bit-exact with the reference
        // (round 0 of a single query: drawn in the kernel prologue)
        if ((round > 0 || first_it <= 0) && (int)tm.lane < CP_N)
            ws.qr[tm.lane] = (float)cp_halton((i64)it + Q.seed_offset, tm.lane);
        tm.sync();
        // _attempt_extend (planner.py:265-306) + commit
        const int node = cp_extend_once(tm, ws, A, sc, Q, qi, a, st);
        if (node == -4) break;
        if (node < 0) continue;
        st.v[ST_ADDED]++;
        // connect the other tree toward q_new (planner.py:463)
        cp_copy(tm, ws.qt, ws.qe);
        const int meet = cp_connect(tm, ws, A, sc, Q, qi, b, st);
        if (meet < 0) continue;
        // junction (planner.py:466-481)
        cp_load_node(tm, A, qi, b, meet, ws.qm);
        const float* js = a == 0 ? ws.qt : ws.qm;
        const float* jg = a == 0 ? ws.qm : ws.qt;
        bool ok = cp_vec_equal(tm, js, jg);
        if (!ok) {
            cp_copy(tm, ws.qr, js);   // derive_edge overwrites seg / qs only
            cp_copy(tm, ws.qn, jg);
            ok = cp_derive_edge(tm, ws, A, sc, ws.qr, ws.qn, st, &Q.stop);
        }
        if (ok) {
            int won = 0;
            if (tm.lane == 0 && atomicCAS(&Q.solved, 0, 1) == 0) {
                Q.meet[a] = node;
                Q.meet[b] = meet;
                Q.t_end_ns = cp_clock_ns();
#ifdef CP_TIMELINE
                Q.pad1_[4] = (int)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
#endif
                // no fence: the stop word is only a signal to leave (the
                // finalizer reads meet / t_end after the active-count handshake)
                atomicExch(&Q.stop, 1);
                // first-solution flag of a race: one store into every racer's word
                for (int r = 0; r < A.n_race; r++) *(volatile int*)A.race_peers[r] = 1;
                if (A.n_race) __threadfence_system();
                won = 1;
            }
            if (tm.bcast(won, 0))   // while the other teams leave
                cp_extract_path(tm, A, qi, a == 0 ? node : meet, a == 0 ? meet : node, ws.seg, nullptr);
            break;
        }
    }
    if (tm.lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_NSTAT; i++)
            if (st.v[i]) atomicAdd(&Q.stats[i], st.v[i]);
    }
}

__host__ __device__ __forceinline__ int cp_pad8(int x) { return (x + CP_CHUNK - 1) / CP_CHUNK * CP_CHUNK; }
__device__ __forceinline__ int cp_scene_f4(const SceneSm& g) {
    return g.cull ? CP_BCH * g.nbc + CP_SCH * g.nec + 2 * ((g.nbc + 7) / 8 + (g.nec + 7) / 8)
                  : 2 * cp_pad8(g.nb) + cp_pad8(g.ne);
}

// One contiguous global -> shared copy by the Tensor Memory Accelerator: a
// single thread issues 1D bulk copies (cp.async.bulk, <= 32 KB each) that
// complete on a shared-memory mbarrier carrying the byte count; every thread
// waits on the barrier's phase (no per-thread loads, no CTA barrier after).
// Up to three blocks (dst[i] <- src[i], bytes[i], multiples of 16) on one barrier.
__device__ __forceinline__ void cp_bulk_to_smem(float4* const* dst, const float4* const* src, const unsigned* bytes,
                                                int nblk) {
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = cp_smem_addr(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned total = 0;
        for (int k = 0; k < nblk; k++) total += bytes[k];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(total) : "memory");
        for (int k = 0; k < nblk; k++) {
            const unsigned d = cp_smem_addr(dst[k]);
            for (unsigned off = 0; off < bytes[k]; off += 32768u) {
                const unsigned n = bytes[k] - off < 32768u ? bytes[k] - off : 32768u;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(d + off), "l"(reinterpret_cast<const char*>(src[k]) + off), "r"(n), "r"(b)
                             : "memory");
            }
        }
    }
    cp_mb_wait(&bar, 0);
}

// Stage the scene into shared memory.  Reference order: padded to whole
// CP_CHUNKs with primitives 1e18 m away (never hit), so the check loop has no
// bounds test.  Clustered: one contiguous block (the host padded the chunks),
// copied by TMA bulk copies.
__device__ __forceinline__ SceneSm cp_stage_scene(const SceneSm& g, float4* sm) {
    SceneSm s = g;
    if (g.cull) {
        const int tot = cp_scene_f4(g);
        if (tot > 0) {
            float4* d[1] = {sm};
            const float4* sr[1] = {g.cl};
            const unsigned n[1] = {(unsigned)tot * 16u};
            cp_bulk_to_smem(d, sr, n, 1);
        }
        s.cl = sm;
        return s;
    }
    const int nbp = cp_pad8(g.nb), nep = cp_pad8(g.ne);
    float4* bc = sm;
    float4* bh = sm + nbp;
    float4* sp = sm + 2 * nbp;
    const float4 far = make_float4(1e18f, 1e18f, 1e18f, 0.f);
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    // the primitives by TMA bulk copies, the chunk padding by the threads
    // (disjoint ranges), then one CTA barrier for the padding stores
    for (int i = g.nb + threadIdx.x; i < nbp; i += blockDim.x) { bc[i] = far; bh[i] = zero; }
    for (int i = g.ne + threadIdx.x; i < nep; i += blockDim.x) sp[i] = far;
    {
        float4* d[3] = {bc, bh, sp};
        const float4* sr[3] = {g.box_c, g.box_h, g.sph};
        const unsigned n[3] = {(unsigned)g.nb * 16u, (unsigned)g.nb * 16u, (unsigned)g.ne * 16u};
        if (g.nb + g.ne > 0) cp_bulk_to_smem(d, sr, n, 3);
    }
    __syncthreads();
    s.box_c = bc; s.box_h = bh; s.sph = sp;
    return s;
}

#if !CP_PARITY
// The solved query's path (planner.py:488-505), by the team that solved it,
// right away -- it overlaps the other teams' exit, but the host waits for it.
// Lanes 0 and 1 walk the start and the goal parent chains concurrently (one
// dependent L2 load per step, meet node first) and every step's two nodes are
// handed to the team by shuffle: chain entry e lives in lane e % CP_G,
// register slot e / CP_G, so reversing the start chain and splicing the goal
// chain is a shuffle per slot, not a round trip through a global index list.
// The team then gathers 16 nodes' coordinates at a time (one round of
// independent L2 loads) into its shared-memory segment rows and writes them
// to the mapped result lane-consecutively (coalesced PCIe writes).  Chains
// longer than the registers hold (CP_XK CP_G entries) take the same walk's
// global index list instead.  meet0 / meet1: the meet nodes in the start /
// goal tree (the winner's registers; also in Q.meet).  setup_code is written
// by cp_check_kernel.
#define CP_XK 4
__device__ __noinline__ void cp_extract_path(const Team tm, const PlanArgs& A, int qi, int meet0, int meet1,
                                             float (*stage)[CP_NP], const PairBox* bx) {
    QueryOut& O = A.out[qi];
    const int lane = (int)tm.lane, cap = A.cap, path_cap = A.path_cap;
    const float* ts = cp_tree(A, qi, 0);
    const float* tg = cp_tree(A, qi, 1);
    const int* ps = cp_par(A, qi, 0);
    const int* pg = cp_par(A, qi, 1);
    int* ch = A.chain + (size_t)qi * path_cap;   // long chains: path position -> (tree << 30) | node
    // the two meet nodes' coordinates (equal: the junction node appears once), in flight during the walk
    const float cm0 = lane < CP_N ? __ldcg(ts + (size_t)lane * cap + meet0) : 0.f;
    const float cm1 = lane < CP_N ? __ldcg(tg + (size_t)lane * cap + meet1) : 0.f;
    // a chain node is visible, so its parent store is issued: a -1 (the reset
    // value) means it has not landed yet -- read again until it has
    auto parent_of = [](const int* pp, int i) {
        int p = cp_ldvol(pp + i);
        while (p < 0) p = cp_ldvol(pp + i);
        return p;
    };
    int rs[CP_XK], rg[CP_XK];   // start / goal chain entries e = CP_G slot + lane
#pragma unroll
    for (int j = 0; j < CP_XK; j++) { rs[j] = 0; rg[j] = 0; }
    int cur = lane == 0 ? meet0 : meet1, cnt = 0;
    bool walking = lane < 2;
    // pair mode: the certifier's ancestor cache of tree `lane` (lanes 0 / 1),
    // when it starts at this chain's meet node (root flag, then length, then entries)
    const int* cc = nullptr;
    int clen = 0, ch0 = 0;
    bool croot = false;
    if (bx && walking) {
        croot = *(const volatile int*)&bx->pw_root[lane] != 0;
        __threadfence_block();
        clen = *(const volatile int*)&bx->pw_len[lane];
        ch0 = *(const volatile int*)&bx->pw_h[lane];
        __threadfence_block();
        if (clen > 0 && bx->pw_anc[lane][ch0] == cur) cc = &bx->pw_anc[lane][ch0];
        else clen = 0;
    }
#ifdef CP_TIMELINE
    const int dbg_clen = clen, dbg_croot = croot ? 1 : 0;
#endif
    if (bx) {   // both chains cached down to their roots: every lane takes its entries from shared memory
        const int l0 = tm.bcast(croot ? clen : 0, 0), l1 = tm.bcast(croot ? clen : 0, 1);
        const int h0 = tm.bcast(ch0, 0), h1 = tm.bcast(ch0, 1);
        if (l0 > 0 && l1 > 0) {   // (a cache holds at most CP_PW <= CP_XK CP_G entries)
#pragma unroll
            for (int j = 0; j < CP_XK; j++) {
                const int e = CP_G * j + lane;
                rs[j] = e < l0 ? bx->pw_anc[0][h0 + e] : 0;
                rg[j] = e < l1 ? bx->pw_anc[1][h1 + e] : 0;
            }
            cnt = lane == 0 ? l0 : l1;
            walking = false;
        }
    }
    for (int c = 0;; c++) {
        const unsigned wm = tm.ballot(walking);
        if (!(wm & 3u) || c > cap) break;   // (a chain is never longer than its tree)
        const int e0 = tm.bcast(cur, 0), e1 = tm.bcast(cur, 1);
        if (c % CP_G == lane) {
#pragma unroll
            for (int j = 0; j < CP_XK; j++)
                if (c / CP_G == j) {
                    if (wm & 1u) rs[j] = e0;
                    if (wm & 2u) rg[j] = e1;
                }
        }
        if (walking) {
            if (c < path_cap) {
                if (lane == 0) ch[c] = cur;                              // start chain, meet first
                else ch[path_cap - 1 - c] = (1 << 30) | cur;             // goal chain, from the end
            }
            cnt++;
            const int p = c + 1 < clen ? cc[c + 1]
                                       : (croot && c + 1 == clen ? cur : parent_of(lane == 0 ? ps : pg, cur));
            if (p == cur) walking = false;
            else cur = p;
        }
    }
    const int ca = tm.bcast(cnt, 0), cb = tm.bcast(cnt, 1);
#ifdef CP_TIMELINE
    {   // diagnostic: cached chain lengths / root flags / chain lengths of both trees
        const int l0 = tm.bcast(dbg_clen, 0), l1 = tm.bcast(dbg_clen, 1);
        const int r0 = tm.bcast(dbg_croot, 0), r1 = tm.bcast(dbg_croot, 1);
        if (lane == 0) A.qs[qi].pad1_[5] = (l0 << 24) | (l1 << 16) | (r0 << 15) | (r1 << 14) | (min(ca, 127) << 7) | min(cb, 127);
    }
#endif
    const int skip = tm.ballot(lane < CP_N && cm0 != cm1) == 0u ? 1 : 0;
    const int len = ca + cb - skip;
    int status = 0;
    if (len > path_cap || ca + cb > path_cap) {
        status = 4;
    } else if (ca <= CP_XK * CP_G && cb <= CP_XK * CP_G) {
        float* path = A.paths + (size_t)qi * path_cap * CP_N;
        for (int base = 0; base < len; base += CP_G) {
            // position k: start chain entry ca - 1 - k, then goal chain entry k - ca + skip
            const int k = base + lane;
            const bool st = k < ca;
            const int e = st ? ca - 1 - k : k - ca + skip;
            int node = 0;
#pragma unroll
            for (int j = 0; j < CP_XK; j++) {
                const int vs = __shfl_sync(tm.mask, rs[j], e % CP_G, CP_G);
                const int vg = __shfl_sync(tm.mask, rg[j], e % CP_G, CP_G);
                if (e / CP_G == j) node = st ? vs : vg;
            }
            if (k < len) {
                const float* t = st ? ts : tg;
#pragma unroll
                for (int d = 0; d < CP_N; d++) stage[lane][d] = __ldcg(t + (size_t)d * cap + node);
            }
            tm.sync();
            const int rows = min(CP_G, len - base);
            for (int f = lane; f < rows * CP_N; f += CP_G) {
                const int r = f / CP_N;
                path[(size_t)base * CP_N + f] = stage[r][f - r * CP_N];
            }
            tm.sync();
        }
    } else {
        // long chains: the global index list, root .. meet .. root
        __threadfence_block();
        tm.sync();
        if (lane == 0) {
            for (int a = 0, b = ca - 1; a < b; a++, b--) { int t = ch[a]; ch[a] = ch[b]; ch[b] = t; }
            for (int k = skip; k < cb; k++) ch[ca + k - skip] = ch[path_cap - 1 - k];
        }
        __threadfence_block();
        tm.sync();
        float* path = A.paths + (size_t)qi * path_cap * CP_N;
        for (int f = lane; f < len * CP_N; f += CP_G) {
            const int k = f / CP_N, d = f - k * CP_N;
            const int e = ch[k];
            path[f] = __ldcg(((e >> 30) ? tg : ts) + (size_t)d * cap + (e & 0x3fffffff));
        }
    }
    if (status == 0) {
        // edge sources: start edges, then the junction (or the first goal
        // edge when the meet nodes coincide), then goal edges
        int* src = A.sources + (size_t)qi * path_cap;
        for (int k = lane; k < len - 1; k += CP_G) src[k] = k < ca - 1 ? 0 : (k == ca - 1 ? (skip ? 2 : 1) : 2);
    }
    if (lane == 0) {
        O.status = status;
        O.path_len = status == 0 ? len : 0;
#ifdef CP_TIMELINE
        QueryState& Q = A.qs[qi];
        Q.pad1_[1] = (int)(cp_clock_ns() - Q.t0_ns);
#endif
    }
    // the path reaches the host before the finalizer's completion word (pair
    // mode: the same lanes finalise next, behind their own system fence)
    if (A.nq == 1 && !A.pair) __threadfence_system();
    tm.sync();
}

// The rest of the result, by the last team to leave the query (when the node
// counts and the stats are final): counters, node counts, device time and,
// for an unsolved query, its status.  setup_code is written by cp_check_kernel.
__device__ __noinline__ void cp_extract_query(const Team tm, const PlanArgs& A, int qi) {
    QueryState& Q = A.qs[qi];
    QueryOut& O = A.out[qi];
    const int lane = (int)tm.lane, cap = A.cap;
    const int ns = min(cp_ldvol(&Q.count[0]), cap), ng = min(cp_ldvol(&Q.count[1]), cap);
#ifndef CP_PROFILE
#ifdef CP_TIMELINE
    if (lane < 6) O.stats[lane] = (u64)cp_ldvol(&Q.pad1_[lane < 5 ? 6 + lane : 13]);   // latest exit by reason
#else
    if (lane < ST_NSTAT) O.stats[lane] = __ldcg(&Q.stats[lane]);
    if (ST_NSTAT > CP_G && lane + CP_G < ST_NSTAT) O.stats[lane + CP_G] = __ldcg(&Q.stats[lane + CP_G]);
#endif
#endif
    const int solved = cp_ldvol(&Q.solved);
    if (lane == 0) {
        if (!solved) {
            O.status = cp_ldvol(&Q.timed_out) ? 1 : (cp_ldvol(&Q.overflow) ? 3 : (cp_ldvol(&Q.race_stopped) ? 5 : 2));
            O.path_len = 0;
        }
        O.n_nodes[0] = ns;
        O.n_nodes[1] = ng;
        Q.hwm[0] = ns;
        Q.hwm[1] = ng;
        const u64 tend = solved ? Q.t_end_ns : cp_clock_ns();
#ifdef CP_TIMELINE   // diagnostic: stats 8-11 = solved / chains walked / path written / last team out (ns after init)
        O.stats[8] = solved ? Q.t_end_ns - Q.t0_ns : 0;
        O.stats[9] = (u64)cp_ldvol(&Q.pad1_[2]);   // latest other P: (ns after solve) & ~15 | phase at the solve
        O.stats[10] = (u64)Q.pad1_[1];
        O.stats[11] = cp_clock_ns() - Q.t0_ns;
        O.stats[6] = (u64)cp_ldvol(&Q.pad1_[0]);   // warp C's longest job across the solve (see the certifier)
        O.stats[7] = (u64)cp_ldvol(&Q.pad1_[5]);   // the winner out
#endif
        O.device_ms = (double)(tend - Q.t0_ns) * 1e-6;
        O.total_ms = (double)(cp_clock_ns() - Q.t0_ns) * 1e-6;
    }
    if (A.nq == 1) {   // single query: every lane's result stores reach the host before the completion word
        __threadfence_system();
        tm.sync();
        if (lane == 0) *(volatile unsigned*)&O.done_seq = (unsigned)A.seeds[A.nq];
    }
    tm.sync();
}

#endif

#if !CP_PARITY
// Dynamic smem: [scene float4s][team workspaces]
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 1)
cp_plan_kernel(const __grid_constant__ PlanArgs A) {
    extern __shared__ float4 cp_smem[];
    if (A.nq == 1 && (int)(threadIdx.x & 31) < CP_N) cp_halton_prefetch((int)(threadIdx.x & 31));
    SceneSm sc = cp_stage_scene(A.scene_g, cp_smem);
    TeamWS* wsa = reinterpret_cast<TeamWS*>(cp_smem + cp_scene_f4(A.scene_g));
    const int team_in_cta = (threadIdx.x >> 5) * (32 / CP_G) + (threadIdx.x & 31) / CP_G;
    // a single query: every team starts on it at once with a static first
    // sample -- team k draws sample k + 1, computed here, before the wait
    // below (the seeds were copied before init ran) -- with no queue / steal
    // round trips, and leaves the kernel after it
#ifdef CP_NO_FASTSTART
    const bool single = false;
#else
    const bool single = A.nq == 1;
#endif
    const int teams_per_cta = A.pair ? (int)(blockDim.x >> 6) : (A.solo ? (int)(blockDim.x >> 5) : (int)blockDim.x / CP_G);
    const int n_teams = (int)gridDim.x * teams_per_cta;
    const int gteam = (int)blockIdx.x * teams_per_cta + (A.pair ? (int)(threadIdx.x >> 6) : team_in_cta / (A.solo ? 32 / CP_G : 1));
    const bool sampler = !(A.solo && (int)(threadIdx.x & 31) >= CP_G) && !(A.pair && ((threadIdx.x >> 5) & 1));
    if (single && sampler && (int)(threadIdx.x % CP_G) < CP_N && gteam < A.max_iterations) {
        const int k = (int)(threadIdx.x % CP_G);
        wsa[team_in_cta].qr[k] = (float)cp_halton((i64)(gteam + 1) + A.seeds[0], k);
    }
    // launched as a programmatic dependent of cp_init_kernel: the scene staging
    // and first samples above overlapped it; query state, trees and queue
    // counters are read only after its writes (a no-op in a plain launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (A.pair) {   // pair mailboxes live in shared memory: set them up before any warp uses one
        for (int w = 2 * threadIdx.x; w < (int)(blockDim.x >> 5); w += 2 * blockDim.x) {
            PairBox* b = cp_pair_box(&wsa[w * (32 / CP_G) + 1]);
            cp_mb_init(&b->full, CP_G);
            cp_mb_init(&b->done, CP_G);
            b->pw_len[0] = 0;
            b->pw_len[1] = 0;
            b->p_ndone = 0;
            b->p_pend = 0;
        }
        __syncthreads();
    }
    // latency mode: one team per warp, so divergent teams never share a warp
    if (A.solo && (int)(threadIdx.x & 31) >= CP_G) return;
    Team tm;
    TeamWS& ws = wsa[team_in_cta];
    // pair mode (solo, CP_G = 16): odd warps certify for the even warp before
    // them; the pair's mailbox is the unused half-team slot of the even warp
    PairBox* bx = nullptr;
    if (A.pair) {
        const int w = threadIdx.x >> 5;
        bx = cp_pair_box(&wsa[(w & ~1) * (32 / CP_G) + 1]);
        if (w & 1) {
            if (A.chk_in_kernel && gteam < 2) cp_pair_endpoint_checks(tm, A, gteam, n_teams);
            cp_pair_certifier(tm, ws, *bx, A, sc);
            asm volatile("cp.async.wait_all;" ::: "memory");   // the last stop-word poll has landed
            return;
        }
    }
    int visits = 0;
    for (;;) {
        int qi = -1;
        int h = 0;
        if (single) {
            if (visits > 0) break;
            qi = 0;
        } else {
        if (tm.lane == 0) h = atomicAdd(A.queue_head, 1);
        h = tm.bcast(h, 0);
        if (h < A.nq) {
            qi = h;
        } else {
            // queue drained: join an unfinished query (work stealing).  The
            // team scans CP_G queries per round (one load latency per round,
            // the three flags of a query loaded in parallel), from a start
            // that spreads the teams.
            int s0 = 0;
            if (tm.lane == 0) s0 = atomicAdd(A.team_counter, 1) % A.nq;
            s0 = tm.bcast(s0, 0);
            for (int base = 0; base < A.nq && qi < 0; base += CP_G) {
                const int j = base + (int)tm.lane;
                bool open = false;
                if (j < A.nq) {
                    QueryState& Q = A.qs[(s0 + j) % A.nq];
                    const int st = cp_ldvol(&Q.stop), so = cp_ldvol(&Q.solved), ex = cp_ldvol(&Q.exhausted);
                    const int sc = cp_ldvol(&Q.setup_code);
                    open = !(st | so | ex) && sc == 0;
                }
                const unsigned mk = tm.ballot(open);
                if (mk) qi = (s0 + base + __ffs(mk) - 1) % A.nq;
            }
        }
        }
        if (qi < 0 || ++visits > 4 * A.nq + 4) break;
        QueryState& Q = A.qs[qi];
        if (tm.lane == 0) atomicAdd(&Q.active, 1);
        const int first = single ? gteam + 1 : 0;
        if (bx) cp_plan_query_pair(tm, ws, wsa[((threadIdx.x >> 5) + 1) * (32 / CP_G)], *bx, A, sc, qi, first, n_teams);
        else cp_plan_query(tm, ws, A, sc, qi, first, n_teams);
        // the last team to leave the query extracts its result (a late
        // joiner may extract again: identical values)
        int last = 0;
#ifdef CP_TIMELINE
        if (tm.lane == 0) {
            const int tnow = (int)(cp_clock_ns() - Q.t0_ns);
            if (cp_ldvol(&Q.pad1_[4]) == (int)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u))) Q.pad1_[5] = tnow;
            else atomicMax(&Q.pad1_[3], tnow);
        }
#endif
        if (tm.lane == 0) {
            __threadfence();
            last = atomicSub(&Q.active, 1) == 1;
        }
        // (pair mode: a solved query was finalised by the team that solved it)
        if (tm.bcast(last, 0) && !(bx && cp_ldvol(&Q.solved))) {
            __threadfence();
            cp_extract_query(tm, A, qi);
        }
    }
    if (bx)   // release the certifier warp
        cp_pair_post(tm, *bx, ws, 0, 0, 0, true, ws.qr, ws.qr, ws.seg, 0, 1);
    asm volatile("cp.async.wait_all;" ::: "memory");   // the last stop-word poll has landed
}

#endif  // !CP_PARITY

// FP64 endpoint test of one configuration (planner.py:416-427
// _check_endpoint): limits, manifold, collision; one warp.

__device__ int cp_check_config_d(const SetupArgs& S, const double* q, int lane, int nl, unsigned mask) {
    // 1 limits, 2 manifold, 3 collision, 0 ok  (evaluated by the nl lanes of mask)
    bool lim = false;
#pragma unroll
    for (int k = 0; k < CP_N; k++) lim |= (q[k] < cp_lo(k) || q[k] > cp_hi(k));
    if (lim) return 1;
    double R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
    double qq[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) qq[k] = q[k];
    cp_fk<double>(qq, R, P, AX, OR, SPH);
    double qe[4], e[CP_M], s = 0.0;
    cp_quat<double>(R + 9 * CP_EE, qe);
    cp_task_err<double>(S.con, P + 3 * CP_EE, qe, e);
#pragma unroll
    for (int i = 0; i < CP_M; i++) s += e[i] * e[i];
    if (!(sqrt(s) < S.tau_task)) return 2;
    bool hit = false;
    const int E = S.nb + S.ne;
    const int total = CP_S * E + CP_P;
    for (int c = lane; c < total; c += nl) {
        double cl;
        if (c < CP_S * E) {
            int si = c / E, pi = c - si * E;
            double x = 0, y = 0, z = 0;
#pragma unroll
            for (int s2 = 0; s2 < CP_S; s2++)
                if (s2 == si) { x = SPH[3 * s2]; y = SPH[3 * s2 + 1]; z = SPH[3 * s2 + 2]; }
            double r = cp_rad(si);
            if (pi < S.nb) {
                const double* lo = S.box_min + 3 * pi;
                const double* hi = S.box_max + 3 * pi;
                double d2 = 0.0, tt;
                if (x < lo[0]) { tt = lo[0] - x; d2 += tt * tt; } else if (x > hi[0]) { tt = x - hi[0]; d2 += tt * tt; }
                if (y < lo[1]) { tt = lo[1] - y; d2 += tt * tt; } else if (y > hi[1]) { tt = y - hi[1]; d2 += tt * tt; }
                if (z < lo[2]) { tt = lo[2] - z; d2 += tt * tt; } else if (z > hi[2]) { tt = z - hi[2]; d2 += tt * tt; }
                cl = sqrt(d2) - r;
            } else {
                const double* oc = S.sph_c + 3 * (pi - S.nb);
                double dx = x - oc[0], dy = y - oc[1], dz = z - oc[2];
                cl = sqrt((dx * dx + dy * dy) + dz * dz) - (r + S.sph_r[pi - S.nb]);
            }
        } else {
            int k = c - CP_S * E;
            int a = cp_pair_a(k), b = cp_pair_b(k);
            double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
#pragma unroll
            for (int s2 = 0; s2 < CP_S; s2++) {
                if (s2 == a) { ax = SPH[3 * s2]; ay = SPH[3 * s2 + 1]; az = SPH[3 * s2 + 2]; }
                if (s2 == b) { bx = SPH[3 * s2]; by = SPH[3 * s2 + 1]; bz = SPH[3 * s2 + 2]; }
            }
            double dx = ax - bx, dy = ay - by, dz = az - bz;
            cl = sqrt((dx * dx + dy * dy) + dz * dz) - (cp_rad(a) + cp_rad(b));
        }
        hit |= cl < 0.0;
    }
    return __any_sync(mask, hit) ? 3 : 0;
}

#if !CP_PARITY
// Per-query state and tree roots (planner.py:442-445); one 32-thread block per
// query.  The NaN refill of the previous run's node slots already happened at
// the end of that run (cp_reset_kernel, outside the timed region).
extern "C" __global__ void __launch_bounds__(32) cp_init_kernel(const __grid_constant__ SetupArgs S) {
    // the planner may start its prologue (scene staging) now; it waits for
    // this grid's writes before touching query state (griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;");
    const int qi = blockIdx.x, lane = threadIdx.x;
    QueryState& Q = S.qs[qi];
    if (qi == 0 && lane < 16 && S.counters) S.counters[lane] = 0;
    if (lane < CP_N) {
        S.trees[((size_t)(2 * qi) * CP_N + lane) * S.cap] = (float)S.starts[(size_t)qi * CP_N + lane];
        S.trees[((size_t)(2 * qi + 1) * CP_N + lane) * S.cap] = (float)S.goals[(size_t)qi * CP_N + lane];
    }
    if (lane == 0) {
        S.parents[(size_t)(2 * qi) * S.cap] = 0;
        S.parents[(size_t)(2 * qi + 1) * S.cap] = 0;
        // stop and setup_code belong to the endpoint checks, which run
        // concurrently (cp_check_kernel); the previous run's cp_reset_kernel
        // cleared them
        Q.seed_offset = S.seeds[qi];
        Q.count[0] = 1; Q.count[1] = 1;
        Q.next_sample = 0;
        Q.solved = 0; Q.timed_out = 0; Q.overflow = 0; Q.exhausted = 0; Q.race_stopped = 0;
        Q.active = 0;
        Q.chk_cnt = 0;
        Q.meet[0] = -1; Q.meet[1] = -1;
        Q.t0_ns = cp_clock_ns();
        Q.t_end_ns = 0;
#ifdef CP_TIMELINE
        Q.pad1_[0] = 0; Q.pad1_[2] = 0; Q.pad1_[3] = 0; Q.pad1_[4] = -1; Q.pad1_[5] = 0;
        for (int k = 6; k < 14; k++) Q.pad1_[k] = 0;
#endif
    }
    if (lane < ST_NSTAT) Q.stats[lane] = 0ull;
}

// FP64 endpoint checks (planner.py:416-427 _check_endpoint), run concurrently
// with the planner (its own graph branch): a bad start / goal stops the query
// and its code goes straight to the results (the host then reports the
// reference's PlanSetupError).  One 64-thread block per query: warp 0 checks
// the start, warp 1 the goal.
extern "C" __global__ void __launch_bounds__(64) cp_check_kernel(const __grid_constant__ SetupArgs S) {
    const int qi = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    QueryState& Q = S.qs[qi];
    __shared__ int codes[2];
    const double* q = (w == 0 ? S.starts : S.goals) + (size_t)qi * CP_N;
    int code = cp_check_config_d(S, q, lane, 32, 0xffffffffu);
    if (lane == 0) codes[w] = code;
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = codes[0] ? codes[0] : (codes[1] ? 3 + codes[1] : 0);
        S.out[qi].setup_code = c;
        if (c) {
            Q.setup_code = c;
            atomicExch(&Q.stop, 1);
        }
        if (gridDim.x == 1) {   // single query: the completion word, with the call's sequence number
            __threadfence_system();
            *(volatile unsigned*)&S.out[qi].chk_seq = (unsigned)S.seeds[gridDim.x];
        }
    }
}

// Reset the node slots used by the previous run to NaN (publication marker),
// and the stop / setup words for the next run's concurrent endpoint checks.
extern "C" __global__ void cp_reset_kernel(QueryState* qs, float* trees, int* parents, int cap, int nq) {
    for (int qk = blockIdx.y; qk < 2 * nq; qk += gridDim.y) {
        const int qi = qk >> 1, k = qk & 1;
        // every slot appended, including by a certifier still finishing its
        // job after the query's finalizer ran (count is final: the planner grid is done)
        const int h = min(max(qs[qi].hwm[k], qs[qi].count[k]), cap);
        if (k == 0 && blockIdx.x == 0 && threadIdx.x == 0) { qs[qi].stop = 0; qs[qi].setup_code = 0; }
        float* base = trees + (size_t)qk * CP_N * cap;
        int* pb = parents + (size_t)qk * cap;
        const float nan = __int_as_float(0x7fffffff);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < h; i += gridDim.x * blockDim.x) {
            pb[i] = -1;
            for (int d = 0; d < CP_N; d++) base[(size_t)d * cap + i] = nan;
        }
    }
}

#endif  // !CP_PARITY
#if CP_PARITY

// ===========================================================================
// Parity / batch entry kernels (one team per item)
// ===========================================================================
template <class T>
__device__ __forceinline__ void cp_fk_item(const double* qin, double* frames, double* axes, double* orgs,
                                           double* ee, double* sph, int i) {
    T q[CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) q[k] = (T)qin[(size_t)i * CP_N + k];
    T R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3];
    cp_fk<T>(q, R, P, AX, OR, SPH);
    if (frames)
        for (int j = 0; j < CP_N; j++) {
            for (int k = 0; k < 9; k++) frames[((size_t)i * CP_N + j) * 12 + k] = R[9 * j + k];
            for (int k = 0; k < 3; k++) frames[((size_t)i * CP_N + j) * 12 + 9 + k] = P[3 * j + k];
        }
    if (axes)
        for (int j = 0; j < 3 * CP_N; j++) { axes[(size_t)i * 3 * CP_N + j] = AX[j]; orgs[(size_t)i * 3 * CP_N + j] = OR[j]; }
    if (ee) {
        T qe[4];
        cp_quat<T>(R + 9 * CP_EE, qe);
        for (int k = 0; k < 3; k++) ee[(size_t)i * 7 + k] = P[3 * CP_EE + k];
        for (int k = 0; k < 4; k++) ee[(size_t)i * 7 + 3 + k] = qe[k];
    }
    if (sph)
        for (int s = 0; s < CP_S; s++) {
            for (int k = 0; k < 3; k++) sph[((size_t)i * CP_S + s) * 4 + k] = SPH[3 * s + k];
            sph[((size_t)i * CP_S + s) * 4 + 3] = cp_rad(s);
        }
}

extern "C" __global__ void cp_fk_kernel(int B, int fp64, const double* q, double* frames, double* axes,
                                        double* orgs, double* ee, double* sph) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    if (fp64) cp_fk_item<double>(q, frames, axes, orgs, ee, sph, i);
    else cp_fk_item<float>(q, frames, axes, orgs, ee, sph, i);
}

template <class T>
__device__ __forceinline__ void cp_tej_item(const Con<T>& c, const double* qin, double* e_out, double* J_out, int i) {
    T q[CP_N], e[CP_M], J[CP_M][CP_N];
#pragma unroll
    for (int k = 0; k < CP_N; k++) q[k] = (T)qin[(size_t)i * CP_N + k];
    cp_err_jac<T>(c, q, e, J);
    for (int r = 0; r < CP_M; r++) {
        e_out[(size_t)i * CP_M + r] = e[r];
        for (int k = 0; k < CP_N; k++) J_out[((size_t)i * CP_M + r) * CP_N + k] = J[r][k];
    }
}

extern "C" __global__ void cp_tej_kernel(int B, int fp64, Con<float> cf, Con<double> cd, const double* q,
                                         double* e, double* J) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    if (fp64) cp_tej_item<double>(cd, q, e, J, i);
    else cp_tej_item<float>(cf, q, e, J, i);
}

// task error at given poses (reference task_error_at), FP64
extern "C" __global__ void cp_err_at_kernel(int B, Con<double> cd, const double* pose, double* e) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    double p[3], qe[4], ee[CP_M];
    for (int k = 0; k < 3; k++) p[k] = pose[(size_t)i * 7 + k];
    for (int k = 0; k < 4; k++) qe[k] = pose[(size_t)i * 7 + 3 + k];
    cp_task_err<double>(cd, p, qe, ee);
    for (int r = 0; r < CP_M; r++) e[(size_t)i * CP_M + r] = ee[r];
}

// Newton projection of single configurations, FP64 (projection.py:231-254)
extern "C" __global__ void cp_project_config_kernel(int B, Con<double> cd, double tau, double lam, int max_iters,
                                                    double* q_io, int* ok_out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    double q[CP_N];
    for (int k = 0; k < CP_N; k++) q[k] = q_io[(size_t)i * CP_N + k];
    int ok = 0;
    for (int it = 0; it < max_iters; it++) {
        bool fin = true;
        for (int k = 0; k < CP_N; k++) fin &= cp_finite(q[k]);
        if (!fin) break;
        double e[CP_M], J[CP_M][CP_N], st[CP_N], s = 0.0;
        cp_err_jac<double>(cd, q, e, J);
        for (int r = 0; r < CP_M; r++) s += e[r] * e[r];
        if (sqrt(s) < tau) {
            double qc[CP_N];
            bool moved = false;
            for (int k = 0; k < CP_N; k++) {
                qc[k] = fmin(fmax(q[k], cp_lo(k)), cp_hi(k));
                moved |= !(qc[k] == q[k]);
            }
            if (!moved) { ok = 1; break; }
            double R[CP_N * 9], P[CP_N * 3], AX[CP_N * 3], OR[CP_N * 3], SPH[(CP_S > 0 ? CP_S : 1) * 3], qe[4], e2[CP_M];
            cp_fk<double>(qc, R, P, AX, OR, SPH);
            cp_quat<double>(R + 9 * CP_EE, qe);
            cp_task_err<double>(cd, P + 3 * CP_EE, qe, e2);
            double s2 = 0.0;
            for (int r = 0; r < CP_M; r++) s2 += e2[r] * e2[r];
            for (int k = 0; k < CP_N; k++) q[k] = qc[k];
            ok = sqrt(s2) < tau;
            break;
        }
        if (!cp_damped<double, CP_M>(J, e, lam, st)) break;
        for (int k = 0; k < CP_N; k++) q[k] = q[k] - st[k];
    }
    for (int k = 0; k < CP_N; k++) q_io[(size_t)i * CP_N + k] = q[k];
    ok_out[i] = ok;
}

// Exact endpoint-style checks for a batch of configurations, FP64:
// 0 ok, 1 limits, 2 manifold, 3 collision.  One warp per configuration.
extern "C" __global__ void cp_check_config_kernel(int B, const __grid_constant__ SetupArgs S, const double* q, int* code) {
    int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= B) return;
    int c = cp_check_config_d(S, q + (size_t)i * CP_N, threadIdx.x & 31, 32, 0xffffffffu);
    if ((threadIdx.x & 31) == 0) code[i] = c;
}

// Batch motion validation with reference semantics (exact counters), or
// (CULL) through the clustered broad phase.  One team per motion; wps
// (B, W, CP_N) FP64 in, scene staged in smem.  Two kernels so that each keeps
// its own register allocation.
template <bool CULL>
__device__ __forceinline__ void cp_validate_batch(int B, int W, int flag_on, float margin, SceneSm scg,
                                                  const double* wps, int* valid, int* first_bad,
                                                  i64* performed, i64* gpu_checks) {
    extern __shared__ float4 cp_smem[];
    scg.cull = CULL ? 1 : 0;   // compile-time layout
    SceneSm sc = cp_stage_scene(scg, cp_smem);
    TeamWS* wsa = reinterpret_cast<TeamWS*>(cp_smem + cp_scene_f4(scg));
    Team tm;
    const int tpc = CP_NTHREADS / CP_G;
    const int team_in_cta = (threadIdx.x >> 5) * (32 / CP_G) + (threadIdx.x & 31) / CP_G;
    TeamWS& ws = wsa[team_in_cta];
    for (int i = blockIdx.x * tpc + team_in_cta; i < B; i += gridDim.x * tpc) {
        tm.sync();
        if ((int)tm.lane < W)
            for (int k = 0; k < CP_N; k++) ws.seg[tm.lane][k] = (float)wps[((size_t)i * W + tm.lane) * CP_N + k];
        tm.sync();
        ValOut o = CULL ? cp_validate_cull(tm, ws.seg, W, 0, flag_on != 0, margin, sc)
                        : cp_validate(tm, ws.seg, W, 0, flag_on != 0, margin, sc);
        if (tm.lane == 0) {
            valid[i] = o.valid;
            first_bad[i] = o.first_bad;
            performed[i] = o.performed;
            if (gpu_checks) gpu_checks[i] = o.gpu_checks;
        }
    }
}
// three resident CTAs per SM (<= 85 registers)
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 3)
cp_validate_kernel(int B, int W, int flag_on, float margin, SceneSm scg, const double* wps, int* valid,
                   int* first_bad, i64* performed, i64* gpu_checks) {
    cp_validate_batch<false>(B, W, flag_on, margin, scg, wps, valid, first_bad, performed, gpu_checks);
}
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 1)
cp_validate_cull_kernel(int B, int W, int flag_on, float margin, SceneSm scg, const double* wps, int* valid,
                        int* first_bad, i64* performed, i64* gpu_checks) {
    cp_validate_batch<true>(B, W, flag_on, margin, scg, wps, valid, first_bad, performed, gpu_checks);
}

// Batch segment projection (parallel / literal-gap / sequential), FP32.
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 1)
cp_project_kernel(int B, int W, Con<float> con, ProjArgs pa, const float* tau_sm, const double* wps, double* xi,
                  int* ok, int* iters, int* prog, float* trace, int* trace_prog) {
    extern __shared__ float4 cp_smem[];
    TeamWS* wsa = reinterpret_cast<TeamWS*>(cp_smem);
    Team tm;
    const int tpc = CP_NTHREADS / CP_G;
    const int team_in_cta = (threadIdx.x >> 5) * (32 / CP_G) + (threadIdx.x & 31) / CP_G;
    TeamWS& ws = wsa[team_in_cta];
    for (int i = blockIdx.x * tpc + team_in_cta; i < B; i += gridDim.x * tpc) {
        tm.sync();
        if ((int)tm.lane < W)
            for (int k = 0; k < CP_N; k++) ws.seg[tm.lane][k] = (float)wps[((size_t)i * W + tm.lane) * CP_N + k];
        tm.sync();
        ProjArgs p = pa;
        if (tau_sm) p.tau_sm_fixed = tau_sm[i];
        int it, pr;
        bool good = cp_project(tm, ws.seg, W, p, &it, &pr,
                               trace ? trace + (size_t)i * pa.max_iters * W * CP_N : nullptr,
                               trace ? trace_prog + (size_t)i * pa.max_iters : nullptr);
        tm.sync();
        // a coordinate the projection left at the FP32 image of its input is
        // returned as the FP64 input itself: row 0 (never rewritten,
        // pure.py:573-574) and every row of a segment that validates at
        // iteration 1 (returned as given, pure.py:569-572 -- e.g. the
        // unconstrained tau = inf sentinel, T/test_projection.py:107-114) come
        // back bit-identical, as in the reference
        if ((int)tm.lane < W)
            for (int k = 0; k < CP_N; k++) {
                const size_t o = ((size_t)i * W + tm.lane) * CP_N + k;
                const double in = wps[o];
                const float v = ws.seg[tm.lane][k];
                xi[o] = v == (float)in ? in : (double)v;
            }
        if (tm.lane == 0) { ok[i] = good; iters[i] = it; prog[i] = pr; }
    }
}

// Batch nearest neighbour over an SoA node array (planner.py:198-201).
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 1)
cp_nearest_kernel(int count, int cap, int n_trees, const float* nodes, int Q, const float* queries, int* idx) {
    Team tm;
    const int tpc = CP_NTHREADS / CP_G;
    const int team_in_cta = (threadIdx.x >> 5) * (32 / CP_G) + (threadIdx.x & 31) / CP_G;
    for (int i = blockIdx.x * tpc + team_in_cta; i < Q; i += gridDim.x * tpc) {
        const float* tree = nodes + (size_t)(i % n_trees) * CP_N * cap;
        int r = cp_nearest(tm, tree, cap, count, queries + (size_t)i * CP_N);
        if (tm.lane == 0) idx[i] = r;
    }
}

// Halton samples, FP64 bit-exact (sampling.py:65-81): out[i] = sample at
// index first + i.
extern "C" __global__ void cp_halton_kernel(int count, i64 first, i64 seed_offset, const double* lo,
                                            const double* hi, double* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    for (int k = 0; k < CP_N; k++) {
        double u = cp_radical_inverse_k(first + i + seed_offset, k);
        out[(size_t)i * CP_N + k] = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), u));
    }
}

#endif  // CP_PARITY

#if !CP_PARITY
// Dense edges of a solved path, re-derived on the device exactly as the
// planner certified them (planner.py:508-523 revalidate_path).  One team per
// edge; nodes (E+1, CP_N) FP32, sources (E): 0 start, 1 junction, 2 goal.
extern "C" __global__ void __launch_bounds__(CP_NTHREADS, 1)
cp_dense_kernel(int E, const __grid_constant__ PlanArgs A, const float* nodes, const int* sources, float* dense,
                int* ok) {
    extern __shared__ float4 cp_smem[];
    SceneSm sc = cp_stage_scene(A.scene_g, cp_smem);
    TeamWS* wsa = reinterpret_cast<TeamWS*>(cp_smem + cp_scene_f4(A.scene_g));
    Team tm;
    const int tpc = CP_NTHREADS / CP_G;
    const int team_in_cta = (threadIdx.x >> 5) * (32 / CP_G) + (threadIdx.x & 31) / CP_G;
    TeamWS& ws = wsa[team_in_cta];
    for (int e = blockIdx.x * tpc + team_in_cta; e < E; e += gridDim.x * tpc) {
        const bool rev = sources[e] == 2;
        const float* x = nodes + (size_t)e * CP_N;
        const float* y = nodes + (size_t)(e + 1) * CP_N;
        tm.sync();
        if ((int)tm.lane < CP_N) {
            ws.qr[tm.lane] = rev ? y[tm.lane] : x[tm.lane];
            ws.qn[tm.lane] = rev ? x[tm.lane] : y[tm.lane];
        }
        tm.sync();
        Stats st;
        bool good = cp_derive_edge(tm, ws, A, sc, ws.qr, ws.qn, st);
        tm.sync();
        if ((int)tm.lane < A.W) {
            int row = rev ? A.W - 1 - (int)tm.lane : (int)tm.lane;
            for (int k = 0; k < CP_N; k++) dense[((size_t)e * A.W + row) * CP_N + k] = ws.seg[tm.lane][k];
        }
        if (tm.lane == 0) ok[e] = good;
    }
}

// One reference extend() or connect() step on tree k of query 0 (the host
// uploaded the tree): op 0 extends toward q, op 1 connects toward q
// (planner.py:317-325, 361-409).  One team, 32 threads.
extern "C" __global__ void __launch_bounds__(32)
cp_step_kernel(const __grid_constant__ PlanArgs A, int op, int k, const float* q, int* out, unsigned long long* stats) {
    extern __shared__ float4 cp_smem[];
    SceneSm sc = cp_stage_scene(A.scene_g, cp_smem);
    TeamWS* wsa = reinterpret_cast<TeamWS*>(cp_smem + cp_scene_f4(A.scene_g));
    if ((int)threadIdx.x >= CP_G) return;
    Team tm;
    TeamWS& ws = wsa[0];
    QueryState& Q = A.qs[0];
    if ((int)tm.lane < CP_N) { ws.qr[tm.lane] = q[tm.lane]; ws.qt[tm.lane] = q[tm.lane]; }
    tm.sync();
    Stats st;
    int r, segs = 0;
    if (op == 0) {
        st.v[ST_ATT]++;
        r = cp_extend_once(tm, ws, A, sc, Q, 0, k, st);
        if (r >= 0) st.v[ST_ADDED]++;
    } else {
        r = cp_connect(tm, ws, A, sc, Q, 0, k, st, &segs);
    }
    if (tm.lane == 0) {
        out[0] = r;
        out[1] = segs;
        out[2] = min(Q.count[k], A.cap);
        for (int i = 0; i < ST_NSTAT; i++) stats[i] = st.v[i];
    }
    asm volatile("cp.async.wait_all;" ::: "memory");   // the last stop-word poll has landed
}
#endif  // !CP_PARITY
