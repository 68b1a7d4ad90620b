// runtime.cpp -- host runtime and C ABI of libcprrtc.so (include/cprrtc.h).
//
// Owns, per context: the CUDA stream, the robot description and its generated
// FK source, NVRTC-compiled modules (one per constraint kind x orientation
// lock x team width, cached on disk as sm_100a cubins), the FP32 scene in
// HBM, the planner's query states and SoA trees, and mapped pinned result
// buffers.  CUDA runtime API (cudart_static) for memory and streams; the
// driver API (module load, launch) is reached through
// cudaGetDriverEntryPoint and NVRTC through dlopen, so the library loads on a
// machine without a GPU driver (the CPU test suite checks its exports).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cprrtc.h"
#include "device/cprrtc_shared.h"

static_assert(sizeof(QueryState) == 384 && offsetof(QueryState, count) == 128 && offsetof(QueryState, stats) == 256,
              "QueryState: polled flags, atomics and stats on separate 128-byte lines");

namespace cprrtc {
std::string codegen_robot(const cprrtc_robot& r, std::string* err);
cudaError_t launch_clearance(int B, int kind, const double* a, const double* b, double* out, cudaStream_t st);
cudaError_t launch_damped_step(int B, int m, int n, const double* J, const double* e, double lam, double* step,
                               int32_t* ok, cudaStream_t st);
}  // namespace cprrtc

namespace {

const char* kDeviceSrc =
#include "device_src.inc"
    ;
const char* kSharedSrc =
#include "shared_src.inc"
    ;

constexpr int kThreads = 256;   // CTA size of every team kernel

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(CPRRTC_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e));      \
    } while (0)

// ---------------------------------------------------------------------------
// driver API entry points (via the runtime; no link-time libcuda dependency)
// ---------------------------------------------------------------------------
struct Driver {
    CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
    CUresult (*moduleUnload)(CUmodule) = nullptr;
    CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**) = nullptr;
    CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
    CUresult (*getErrorString)(CUresult, const char**) = nullptr;
    CUresult (*moduleGetGlobal)(CUdeviceptr*, size_t*, CUmodule, const char*) = nullptr;
    CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

Driver& drv() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = entry("cuModuleLoadData", d.moduleLoadData) && entry("cuModuleUnload", d.moduleUnload) &&
               entry("cuModuleGetFunction", d.moduleGetFunction) && entry("cuLaunchKernel", d.launchKernel) &&
               entry("cuFuncSetAttribute", d.funcSetAttribute) &&
               entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.occupancy) &&
               entry("cuGetErrorString", d.getErrorString) && entry("cuModuleGetGlobal", d.moduleGetGlobal) &&
               entry("cuLaunchKernelEx", d.launchKernelEx);
    });
    return d;
}

std::string cu_err(CUresult r) {
    const char* s = nullptr;
    if (drv().getErrorString) drv().getErrorString(r, &s);
    return s ? s : ("CUresult " + std::to_string((int)r));
}

// ---------------------------------------------------------------------------
// NVRTC (dlopen)
// ---------------------------------------------------------------------------
struct Nvrtc {
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*logSize)(nvrtcProgram, size_t*);
    nvrtcResult (*log)(nvrtcProgram, char*);
    nvrtcResult (*cubinSize)(nvrtcProgram, size_t*);
    nvrtcResult (*cubin)(nvrtcProgram, char*);
    nvrtcResult (*destroy)(nvrtcProgram*);
    nvrtcResult (*version)(int*, int*);
    const char* (*errstr)(nvrtcResult);
    bool ok = false;
    std::string why;
};

Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("cannot load libnvrtc: ") + dlerror();
            return;
        }
#define SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
        SYM(create, "nvrtcCreateProgram");
        SYM(compile, "nvrtcCompileProgram");
        SYM(logSize, "nvrtcGetProgramLogSize");
        SYM(log, "nvrtcGetProgramLog");
        SYM(cubinSize, "nvrtcGetCUBINSize");
        SYM(cubin, "nvrtcGetCUBIN");
        SYM(destroy, "nvrtcDestroyProgram");
        SYM(version, "nvrtcVersion");
        SYM(errstr, "nvrtcGetErrorString");
#undef SYM
        n.ok = n.create && n.compile && n.logSize && n.log && n.cubinSize && n.cubin && n.destroy && n.version &&
               n.errstr;
        if (!n.ok) n.why = "libnvrtc is missing symbols";
    });
    return n;
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string lib_dir() {
    Dl_info info;
    if (dladdr(reinterpret_cast<void*>(&lib_dir), &info) && info.dli_fname) {
        std::string p(info.dli_fname);
        size_t k = p.rfind('/');
        if (k != std::string::npos) return p.substr(0, k);
    }
    return ".";
}

std::string cache_dir() {
    const char* e = getenv("CPRRTC_CACHE_DIR");
    std::string d = e && *e ? e : lib_dir() + "/_nvrtc_cache";
    mkdir(d.c_str(), 0755);
    return d;
}

const char* kArch = "--gpu-architecture=sm_100a";

// Compile (or fetch from the disk cache) a cubin for source `src`.
int nvrtc_cubin(const std::string& src, const std::string& name, std::vector<char>* cubin, std::string* path_out) {
    Nvrtc& nv = nvrtc();
    if (!nv.ok) return fail(CPRRTC_ENVRTC, nv.why);
    int maj = 0, min = 0;
    nv.version(&maj, &min);
    // FP32 division / sqrt approximate (2 ulp) and denormals flushed: the FP32
    // planner has explicit tolerance margins; FP64 code is unaffected
    std::vector<const char*> opts = {kArch, "-std=c++17", "-lineinfo", "-default-device", "--dopt=on",
                                     "--extra-device-vectorization", "-ftz=true", "-prec-div=false",
                                     "-prec-sqrt=false"};
    std::string key = src + "|" + std::to_string(maj) + "." + std::to_string(min);
    for (auto o : opts) key += std::string("|") + o;
    char hex[32];
    std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key));
    std::string path = cache_dir() + "/" + name + "-" + hex + ".cubin";
    if (path_out) *path_out = path;
    {
        std::ifstream f(path, std::ios::binary);
        if (f) {
            cubin->assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
            if (!cubin->empty()) return 0;
        }
    }
    nvrtcProgram prog;
    nvrtcResult r = nv.create(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(CPRRTC_ENVRTC, std::string("nvrtcCreateProgram: ") + nv.errstr(r));
    r = nv.compile(prog, (int)opts.size(), opts.data());
    size_t ls = 0;
    nv.logSize(prog, &ls);
    std::string logtxt(ls, '\0');
    if (ls) nv.log(prog, &logtxt[0]);
    if (r != NVRTC_SUCCESS) {
        nv.destroy(&prog);
        return fail(CPRRTC_ENVRTC, "NVRTC compile failed:\n" + logtxt);
    }
    size_t cs = 0;
    nv.cubinSize(prog, &cs);
    cubin->resize(cs);
    nv.cubin(prog, cubin->data());
    nv.destroy(&prog);
    std::string tmp = path + ".tmp" + std::to_string(getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        f.write(cubin->data(), (std::streamsize)cubin->size());
    }
    std::rename(tmp.c_str(), path.c_str());
    return 0;
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int ensure(size_t need) {
        if (need <= bytes && p) return 0;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t b = need < 256 ? 256 : need;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        bytes = b;
        return 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct HostBuf {   // pinned, mapped
    void* h = nullptr;
    void* d = nullptr;
    size_t bytes = 0;
    ~HostBuf() {
        if (h) cudaFreeHost(h);
    }
    int ensure(size_t need) {
        if (need <= bytes && h) return 0;
        if (h) cudaFreeHost(h);
        h = d = nullptr;
        bytes = 0;
        size_t b = need < 256 ? 256 : need;
        cudaError_t e = cudaHostAlloc(&h, b, cudaHostAllocMapped);
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        e = cudaHostGetDevicePointer(&d, h, 0);
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("cudaHostGetDevicePointer: ") + cudaGetErrorString(e));
        bytes = b;
        return 0;
    }
    template <class T> T* host() const { return static_cast<T*>(h); }
    template <class T> T* dev() const { return static_cast<T*>(d); }
};

struct Module {
    CUmodule mod = nullptr;
    int G = 16, kind = 0, orient = 0;
    size_t ws_bytes = 0;   // sizeof(TeamWS)
    std::map<std::string, CUfunction> fn;
    int plan_occ = 0;      // resident plan CTAs per SM
    std::string cubin_path;
    CUdeviceptr conf_ptr = 0;   // __constant__ Con<float> cp_conf
    Con<float> conf_now{};
    bool conf_valid = false;
};

struct Ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    int n = 0, S = 0, P = 0, NP = 0;
    std::string robot_src;
    std::vector<double> lo, hi;
    // scene
    int nb = 0, ne = 0;
    DevBuf sc_box_c, sc_box_h, sc_sph, sc_bmin, sc_bmax, sc_sc, sc_sr;
    DevBuf sc_cl;          // clustered layout (broad phase), see SceneSm
    DevBuf race_flag;      // first-solution word of cprrtc_plan_race
    int* race_host = nullptr;   // fallback first-solution word without peer access (mapped, portable)
    int nbc = 0, nec = 0;
    // constraint
    int kind = 0, orient = 0;
    Con<float> conf{};
    Con<double> cond{};
    double tau_task = INFINITY;
    std::map<std::tuple<int, int, int, int>, std::unique_ptr<Module>> modules;
    // planner buffers
    int nq_alloc = 0, cap_alloc = 0;
    DevBuf qs, trees, parents, counters, d_starts, d_goals, d_seeds;
    HostBuf h_in, h_out, h_paths, h_src;
    int path_cap = 0;
    PlanArgs last_args{};
    Module* last_mod = nullptr;
    int last_nq = 0;
    DevBuf dense_buf, dense_ok, dense_nodes;
    DevBuf chain;          // path extraction: node index per path position
    // scratch for parity/batch entry points
    DevBuf scratch[10];
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t stream2 = nullptr;          // the endpoint-check branch of the plan graph
    cudaEvent_t fork = nullptr, join = nullptr;
    // cached CUDA graphs of the per-call plan sequence (H2D, setup, plan, extract)
    struct PlanGraph {
        cudaGraphExec_t exec = nullptr;
        PlanArgs A{};
        SetupArgs S{};
        int B = 0, grid = 0, block = 0, path_cap = 0;
        size_t smem = 0;
        Module* m = nullptr;
    };
    std::vector<PlanGraph> graphs;
    double last_total_ms = 0, last_plan_ms = 0;
    bool plan_ev = true;           // ev[1..2] bracket the plan kernel in the current graph
    bool plan_lean = false;        // the current graph is the lean single-query one (no events, no check kernel)
    double last_kernel_total_ms = 0;   // lean graph: init -> last team out (globaltimer)
    double last_query_ms = 0.0;    // longest query device time of the last plan call
    bool timing_pending = false;   // last_*_ms still to be read from ev[0..3] (last plan call)
    int inflight = 0;              // B of a batch submitted and not yet waited for (cprrtc_plan_submit)
    unsigned plan_seq = 0;         // sequence number of the last plan launch (QueryOut completion words)
    int64_t launches = 0;
};

int set_device(Ctx* c) {
    CUDA_TRY(cudaSetDevice(c->device));
    return 0;
}

std::string prelude(const Ctx* c, int G, int kind, int orient, int parity) {
    std::ostringstream os;
    os << "#define CP_G " << G << "\n#define CP_KIND " << kind << "\n#define CP_ORIENT " << orient
       << "\n#define CP_NTHREADS " << kThreads << "\n#define CP_PARITY " << parity << "\n";
    // developer knob for same-box A/B runs: CPRRTC_DEFINES="NAME=VAL,NAME2" adds
    // #defines to every module (and so to the cubin cache key)
    if (const char* d = getenv("CPRRTC_DEFINES")) {
        std::string all(d), item;
        std::stringstream ss(all);
        while (std::getline(ss, item, ',')) {
            if (item.empty()) continue;
            const size_t eq = item.find('=');
            os << "#define " << (eq == std::string::npos ? item : item.substr(0, eq) + " " + item.substr(eq + 1))
               << "\n";
        }
    }
    os << kSharedSrc << "\n" << c->robot_src << "\n";
    return os.str();
}

const std::vector<const char*> kPlanKernels = {"cp_plan_kernel", "cp_init_kernel", "cp_check_kernel",
                                                "cp_reset_kernel", "cp_dense_kernel", "cp_step_kernel"};
const std::vector<const char*> kParityKernels = {"cp_fk_kernel",           "cp_tej_kernel",
                                                  "cp_err_at_kernel",       "cp_project_config_kernel",
                                                  "cp_check_config_kernel", "cp_validate_kernel",
                                                  "cp_validate_cull_kernel", "cp_project_kernel",
                                                  "cp_nearest_kernel",      "cp_halton_kernel"};

std::string module_name(int G, int kind, int orient, int parity) {
    char name[64];
    std::snprintf(name, sizeof name, "cprrtc-%s-g%d-k%d-o%d", parity ? "parity" : "plan", G, kind, orient);
    return name;
}

int get_module(Ctx* c, int G, int kind, int orient, int parity, Module** out) {
    auto key = std::make_tuple(G, kind, orient, parity);
    auto it = c->modules.find(key);
    if (it != c->modules.end()) {
        *out = it->second.get();
        return 0;
    }
    if (!drv().ok) return fail(CPRRTC_ECUDA, "CUDA driver entry points unavailable");
    std::string src = prelude(c, G, kind, orient, parity) + kDeviceSrc;
    std::vector<char> cubin;
    auto m = std::make_unique<Module>();
    int rc = nvrtc_cubin(src, module_name(G, kind, orient, parity), &cubin, &m->cubin_path);
    if (rc) return rc;
    CUresult r = drv().moduleLoadData(&m->mod, cubin.data());
    if (r != CUDA_SUCCESS) return fail(CPRRTC_ECUDA, "cuModuleLoadData: " + cu_err(r));
    for (const char* k : parity ? kParityKernels : kPlanKernels) {
        CUfunction f;
        r = drv().moduleGetFunction(&f, m->mod, k);
        if (r != CUDA_SUCCESS) return fail(CPRRTC_ECUDA, std::string("cuModuleGetFunction ") + k + ": " + cu_err(r));
        m->fn[k] = f;
    }
    {
        size_t sz = 0;
        r = drv().moduleGetGlobal(&m->conf_ptr, &sz, m->mod, "cp_conf");
        if (r != CUDA_SUCCESS || sz != sizeof(Con<float>))
            return fail(CPRRTC_ECUDA, "cp_conf symbol missing or mis-sized: " + cu_err(r));
    }
    m->G = G;
    m->kind = kind;
    m->orient = orient;
    // sizeof(TeamWS): the poll slots (48 B), G segment rows and 7 vectors, 16-byte aligned
    m->ws_bytes = ((size_t)64 + (size_t)(G + 7) * c->NP * sizeof(float) + 15) & ~(size_t)15;
    for (const char* k : {"cp_plan_kernel", "cp_validate_kernel", "cp_validate_cull_kernel", "cp_project_kernel",
                          "cp_dense_kernel", "cp_step_kernel"})
        if (m->fn.count(k)) drv().funcSetAttribute(m->fn[k], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 200 * 1024);
    *out = m.get();
    c->modules[key] = std::move(m);
    return 0;
}

int cur_module(Ctx* c, int W, int parity, Module** m) {
    if (W < 2 || W > 32) return fail(CPRRTC_ELIMIT, "width must be in [2, 32] for this build");
    return get_module(c, W <= 16 ? 16 : 32, c->kind, c->orient, parity, m);
}

// make the module's constant-memory constraint equal to the context's
int upload_conf(Ctx* c, Module* m) {
    if (m->conf_valid && std::memcmp(&m->conf_now, &c->conf, sizeof(Con<float>)) == 0) return 0;
    CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<void*>(m->conf_ptr), &c->conf, sizeof(Con<float>),
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));   // the source is a context member
    m->conf_now = c->conf;
    m->conf_valid = true;
    return 0;
}

int launch(Ctx* c, Module* m, const char* k, unsigned gx, unsigned gy, unsigned bx, size_t smem, void** args,
           cudaStream_t st = nullptr) {
    CUresult r = drv().launchKernel(m->fn[k], gx, gy, 1, bx, 1, 1, (unsigned)smem, (CUstream)(st ? st : c->stream),
                                    args, nullptr);
    if (r != CUDA_SUCCESS) return fail(CPRRTC_ECUDA, std::string("launch ") + k + ": " + cu_err(r));
    c->launches++;
    return 0;
}

// launch as a programmatic dependent of the previous kernel in the stream: it
// may start once that kernel's blocks have all issued griddepcontrol.launch_dependents
int launch_pdl(Ctx* c, Module* m, const char* k, unsigned gx, unsigned bx, size_t smem, void** args) {
    CUlaunchAttribute at[1];
    at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    at[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg = {};
    cfg.gridDimX = gx; cfg.gridDimY = 1; cfg.gridDimZ = 1;
    cfg.blockDimX = bx; cfg.blockDimY = 1; cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)c->stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUresult r = drv().launchKernelEx(&cfg, m->fn[k], args, nullptr);
    if (r != CUDA_SUCCESS) return fail(CPRRTC_ECUDA, std::string("launch ") + k + ": " + cu_err(r));
    c->launches++;
    return 0;
}

int sync(Ctx* c) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("kernel failed: ") + cudaGetErrorString(e));
    return 0;
}

template <class T> int upload(Ctx* c, DevBuf& b, const T* src, size_t count) {
    if (int rc = b.ensure(count * sizeof(T) + 16)) return rc;
    if (count) CUDA_TRY(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    return 0;
}
template <class T> int download(Ctx* c, T* dst, const DevBuf& b, size_t count) {
    if (count) CUDA_TRY(cudaMemcpyAsync(dst, b.p, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

SceneSm scene_args(Ctx* c, int cull = 0) {
    SceneSm s;
    std::memset(&s, 0, sizeof s);
    s.box_c = c->sc_box_c.as<float4>();
    s.box_h = c->sc_box_h.as<float4>();
    s.sph = c->sc_sph.as<float4>();
    s.nb = c->nb;
    s.ne = c->ne;
    s.cl = c->sc_cl.as<float4>();
    s.nbc = c->nbc;
    s.nec = c->nec;
    s.cull = cull ? 1 : 0;
    return s;
}

int pad8(int x) { return (x + 7) / 8 * 8; }

// float4s staged per CTA (cp_scene_f4 in the device code)
size_t scene_f4(int nb, int ne, int nbc, int nec, int cull) {
    return cull ? (size_t)(18 * nbc + 10 * nec + 2 * ((nbc + 7) / 8 + (nec + 7) / 8)) : (size_t)(2 * pad8(nb) + pad8(ne));
}
size_t scene_smem(Ctx* c, int cull = 0) { return scene_f4(c->nb, c->ne, c->nbc, c->nec, cull) * sizeof(float4); }

// Clustered scene (broad phase): primitives sorted along a 30-bit Morton
// curve of their centres, cut into chunks of 8, each chunk led by a bounding
// box rounded outward (FP64 -> FP32 with 1e-5 m + 1e-6 relative slack) so the
// FP32 chunk test can never reject a primitive the FP32 narrow test would hit.
static void build_clusters(const cprrtc_scene* s, std::vector<float4>& out, int& nbc, int& nec) {
    const int nb = s->n_boxes, ne = s->n_spheres;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    auto centre = [&](int kind, int i, int a) {
        return kind == 0 ? 0.5 * (s->box_min[3 * i + a] + s->box_max[3 * i + a]) : s->sph_center[3 * i + a];
    };
    for (int kind = 0; kind < 2; kind++)
        for (int i = 0; i < (kind ? ne : nb); i++)
            for (int a = 0; a < 3; a++) {
                lo[a] = std::min(lo[a], centre(kind, i, a));
                hi[a] = std::max(hi[a], centre(kind, i, a));
            }
    auto spread = [](uint32_t v) {   // 10 bits -> every third bit
        uint64_t x = v & 1023u;
        x = (x | (x << 16)) & 0x030000FFull;
        x = (x | (x << 8)) & 0x0300F00Full;
        x = (x | (x << 4)) & 0x030C30C3ull;
        x = (x | (x << 2)) & 0x09249249ull;
        return x;
    };
    auto morton = [&](int kind, int i) {
        uint64_t code = 0;
        for (int a = 0; a < 3; a++) {
            double ext = hi[a] - lo[a];
            double u = ext > 0 ? (centre(kind, i, a) - lo[a]) / ext : 0.0;
            uint32_t v = (uint32_t)std::min(1023.0, std::max(0.0, u * 1023.0));
            code |= spread(v) << a;
        }
        return code;
    };
    auto bound = [](const double* blo, const double* bhi, float4& c, float4& h) {
        float cc[3], hh[3];
        for (int a = 0; a < 3; a++) {
            double cd = 0.5 * (blo[a] + bhi[a]), hd = 0.5 * (bhi[a] - blo[a]);
            cc[a] = (float)cd;
            hh[a] = (float)((hd + std::fabs(cd - (double)cc[a])) * (1.0 + 1e-6) + 1e-5);
        }
        c = make_float4(cc[0], cc[1], cc[2], 0.f);
        h = make_float4(hh[0], hh[1], hh[2], 0.f);
    };
    const float4 far = make_float4(1e18f, 1e18f, 1e18f, 0.f);
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    out.clear();
    // superchunk bounds (groups of 8 chunks = 64 primitives), appended after
    // the chunks: [box groups (c, h)] [sphere groups (c, h)]
    std::vector<float4> groups[2];
    for (int kind = 0; kind < 2; kind++) {
        const int n = kind ? ne : nb;
        std::vector<std::pair<uint64_t, int>> ord(n);
        for (int i = 0; i < n; i++) ord[i] = {morton(kind, i), i};
        std::sort(ord.begin(), ord.end());
        const int chunks = (n + 7) / 8;
        double glo[3], ghi[3];
        for (int k = 0; k < chunks; k++) {
            if (k % 8 == 0)
                for (int d = 0; d < 3; d++) { glo[d] = INFINITY; ghi[d] = -INFINITY; }
            double blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
            std::vector<float4> a(8), b(8);
            for (int j = 0; j < 8; j++) {
                const int o = 8 * k + j;
                if (o >= n) { a[j] = far; b[j] = zero; continue; }
                const int i = ord[o].second;
                for (int d = 0; d < 3; d++) {
                    double l = kind ? s->sph_center[3 * i + d] - s->sph_radius[i] : s->box_min[3 * i + d];
                    double u = kind ? s->sph_center[3 * i + d] + s->sph_radius[i] : s->box_max[3 * i + d];
                    blo[d] = std::min(blo[d], l);
                    bhi[d] = std::max(bhi[d], u);
                }
                if (kind == 0) {
                    const double* l = s->box_min + 3 * i;
                    const double* u = s->box_max + 3 * i;
                    a[j] = make_float4((float)(0.5 * (l[0] + u[0])), (float)(0.5 * (l[1] + u[1])),
                                       (float)(0.5 * (l[2] + u[2])), 0.f);
                    b[j] = make_float4((float)(0.5 * (u[0] - l[0])), (float)(0.5 * (u[1] - l[1])),
                                       (float)(0.5 * (u[2] - l[2])), 0.f);
                } else {
                    a[j] = make_float4((float)s->sph_center[3 * i], (float)s->sph_center[3 * i + 1],
                                       (float)s->sph_center[3 * i + 2], (float)s->sph_radius[i]);
                }
            }
            float4 c, h;
            bound(blo, bhi, c, h);
            out.push_back(c);
            out.push_back(h);
            for (int j = 0; j < 8; j++) out.push_back(a[j]);
            if (kind == 0)
                for (int j = 0; j < 8; j++) out.push_back(b[j]);
            for (int d = 0; d < 3; d++) { glo[d] = std::min(glo[d], blo[d]); ghi[d] = std::max(ghi[d], bhi[d]); }
            if (k % 8 == 7 || k == chunks - 1) {
                float4 gc, gh;
                bound(glo, ghi, gc, gh);
                groups[kind].push_back(gc);
                groups[kind].push_back(gh);
            }
        }
        (kind ? nec : nbc) = chunks;
    }
    out.insert(out.end(), groups[0].begin(), groups[0].end());
    out.insert(out.end(), groups[1].begin(), groups[1].end());
}

size_t team_smem(Ctx* c, Module* m, bool with_scene) {
    size_t sc = with_scene ? std::max(scene_smem(c, 0), scene_smem(c, 1)) : 0;
    return sc + (size_t)(kThreads / m->G) * m->ws_bytes;
}

float tau_dev(double tau) {
    if (!std::isfinite(tau)) return INFINITY;
    double d = tau * (1.0 - 1e-3) - 2e-6;
    if (d < 0.5 * tau) d = 0.5 * tau;
    return (float)d;
}

Ctx* C(void* p) { return static_cast<Ctx*>(p); }

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int cprrtc_abi_version(void) { return CPRRTC_ABI_VERSION; }

const char* cprrtc_last_error(void) { return g_err.c_str(); }

int cprrtc_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    *count = e == cudaSuccess ? n : 0;
    if (e != cudaSuccess) return fail(CPRRTC_ENODEV, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    return 0;
}

int cprrtc_codegen(const cprrtc_robot* robot, char* buf, size_t cap, size_t* needed) {
    if (!robot) return fail(CPRRTC_EARG, "robot is NULL");
    std::string err;
    std::string s = cprrtc::codegen_robot(*robot, &err);
    if (s.empty()) return fail(CPRRTC_EARG, err);
    if (needed) *needed = s.size() + 1;
    if (buf && cap) {
        size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(buf, s.data(), k);
        buf[k] = '\0';
    }
    return 0;
}

int cprrtc_precompile(const cprrtc_robot* robot, int G, int kind, int orient, int parity, char* path, size_t cap) {
    if (!robot || (G != 16 && G != 32) || (kind != 0 && kind != 1)) return fail(CPRRTC_EARG, "bad argument");
    std::string err;
    Ctx tmp;
    tmp.robot_src = cprrtc::codegen_robot(*robot, &err);
    if (tmp.robot_src.empty()) return fail(CPRRTC_EARG, err);
    std::string src = prelude(&tmp, G, kind, orient ? 1 : 0, parity ? 1 : 0) + kDeviceSrc;
    std::vector<char> cubin;
    std::string where;
    if (int rc = nvrtc_cubin(src, module_name(G, kind, orient ? 1 : 0, parity ? 1 : 0), &cubin, &where)) return rc;
    if (path && cap) {
        std::snprintf(path, cap, "%s", where.c_str());
    }
    return 0;
}

int cprrtc_device_source(const cprrtc_robot* robot, int G, int kind, int orient, int parity, char* buf, size_t cap,
                         size_t* needed) {
    if (!robot) return fail(CPRRTC_EARG, "bad argument");
    std::string err;
    Ctx tmp;
    tmp.robot_src = cprrtc::codegen_robot(*robot, &err);
    if (tmp.robot_src.empty()) return fail(CPRRTC_EARG, err);
    std::string src = prelude(&tmp, G, kind, orient ? 1 : 0, parity ? 1 : 0) + kDeviceSrc;
    if (needed) *needed = src.size() + 1;
    if (buf && cap) {
        size_t k = src.size() < cap - 1 ? src.size() : cap - 1;
        std::memcpy(buf, src.data(), k);
        buf[k] = 0;
    }
    return 0;
}

int cprrtc_ctx_create(int device, const cprrtc_robot* robot, void** out) {
    if (!robot || !out) return fail(CPRRTC_EARG, "NULL argument");
    std::string err;
    std::string src = cprrtc::codegen_robot(*robot, &err);
    if (src.empty()) return fail(CPRRTC_EARG, err);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CPRRTC_ENODEV, "no CUDA device visible (the B200 planner has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(CPRRTC_EARG, "device index out of range");
    auto c = std::make_unique<Ctx>();
    c->device = device;
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(CPRRTC_ENODEV, std::string("sm_100a build needs a Blackwell B200, found ") + prop.name);
    c->sms = prop.multiProcessorCount;
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
    for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
    c->n = robot->n;
    c->S = robot->n_spheres;
    c->P = robot->n_pairs;
    c->NP = (c->n % 2) ? c->n : c->n + 1;
    c->robot_src = src;
    c->lo.assign(robot->lo, robot->lo + robot->n);
    c->hi.assign(robot->hi, robot->hi + robot->n);
    if (!drv().ok) return fail(CPRRTC_ECUDA, "CUDA driver entry points unavailable");
    // unconstrained until told otherwise
    if (int rc = cprrtc_set_constraint(c.get(), nullptr)) return rc;
    cprrtc_scene empty{};
    if (int rc = cprrtc_set_scene(c.get(), &empty)) return rc;
    *out = c.release();
    return 0;
}

int cprrtc_ctx_destroy(void* p) {
    Ctx* c = C(p);
    if (!c) return 0;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->modules)
        if (kv.second->mod) drv().moduleUnload(kv.second->mod);
    for (auto& g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    if (c->stream2) cudaStreamDestroy(c->stream2);
    if (c->race_host) cudaFreeHost(c->race_host);
    cudaStreamDestroy(c->stream);
    delete c;
    return 0;
}

int cprrtc_set_scene(void* p, const cprrtc_scene* s) {
    Ctx* c = C(p);
    if (!c || !s) return fail(CPRRTC_EARG, "NULL argument");
    if (s->n_boxes < 0 || s->n_spheres < 0) return fail(CPRRTC_EARG, "negative primitive count");
    if (scene_f4(s->n_boxes, s->n_spheres, (s->n_boxes + 7) / 8, (s->n_spheres + 7) / 8, 1) * 16 > 180 * 1024)
        return fail(CPRRTC_ELIMIT, "scene exceeds the shared-memory staging capacity (~5000 boxes)");
    if (int rc = set_device(c)) return rc;
    std::vector<float4> bc(s->n_boxes), bh(s->n_boxes), sp(s->n_spheres);
    for (int i = 0; i < s->n_boxes; i++) {
        const double* lo = s->box_min + 3 * i;
        const double* hi = s->box_max + 3 * i;
        bc[i] = make_float4((float)(0.5 * (lo[0] + hi[0])), (float)(0.5 * (lo[1] + hi[1])),
                            (float)(0.5 * (lo[2] + hi[2])), 0.f);
        bh[i] = make_float4((float)(0.5 * (hi[0] - lo[0])), (float)(0.5 * (hi[1] - lo[1])),
                            (float)(0.5 * (hi[2] - lo[2])), 0.f);
    }
    for (int i = 0; i < s->n_spheres; i++)
        sp[i] = make_float4((float)s->sph_center[3 * i], (float)s->sph_center[3 * i + 1],
                            (float)s->sph_center[3 * i + 2], (float)s->sph_radius[i]);
    int rc = upload(c, c->sc_box_c, bc.data(), bc.size());
    rc = rc ? rc : upload(c, c->sc_box_h, bh.data(), bh.size());
    rc = rc ? rc : upload(c, c->sc_sph, sp.data(), sp.size());
    rc = rc ? rc : upload(c, c->sc_bmin, s->box_min, 3 * (size_t)s->n_boxes);
    rc = rc ? rc : upload(c, c->sc_bmax, s->box_max, 3 * (size_t)s->n_boxes);
    rc = rc ? rc : upload(c, c->sc_sc, s->sph_center, 3 * (size_t)s->n_spheres);
    rc = rc ? rc : upload(c, c->sc_sr, s->sph_radius, (size_t)s->n_spheres);
    int nbc = 0, nec = 0;
    std::vector<float4> cl;
    build_clusters(s, cl, nbc, nec);
    rc = rc ? rc : upload(c, c->sc_cl, cl.data(), cl.size());
    if (rc) return rc;
    c->nb = s->n_boxes;
    c->ne = s->n_spheres;
    c->nbc = nbc;
    c->nec = nec;
    return sync(c);
}

int cprrtc_set_constraint(void* p, const cprrtc_constraint* k) {
    Ctx* c = C(p);
    if (!c) return fail(CPRRTC_EARG, "NULL context");
    cprrtc_constraint u{};
    if (!k) {   // unconstrained(): plane z = 0 with tau = inf (constraints.py:179-186)
        u.kind = 0;
        u.anchor[2] = 1.0;
        u.q_fixed[0] = 1.0;
        u.r_fixed_t[0] = u.r_fixed_t[4] = u.r_fixed_t[8] = 1.0;
        u.weight = 0.5;
        u.tau_task = INFINITY;
        k = &u;
    }
    if (k->kind != 0 && k->kind != 1) return fail(CPRRTC_EARG, "constraint kind must be 0 (plane) or 1 (line)");
    c->kind = k->kind;
    c->orient = k->has_orient ? 1 : 0;
    c->tau_task = k->tau_task;
    for (int i = 0; i < 3; i++) {
        c->cond.anchor[i] = k->anchor[i];
        c->cond.b1[i] = k->basis[i];
        c->cond.b2[i] = k->basis[3 + i];
    }
    c->cond.offset = k->offset;
    for (int i = 0; i < 4; i++) c->cond.qf[i] = k->q_fixed[i];
    for (int i = 0; i < 9; i++) c->cond.rft[i] = k->r_fixed_t[i];
    c->cond.weight = k->weight;
    for (int i = 0; i < 3; i++) {
        c->conf.anchor[i] = (float)c->cond.anchor[i];
        c->conf.b1[i] = (float)c->cond.b1[i];
        c->conf.b2[i] = (float)c->cond.b2[i];
    }
    c->conf.offset = (float)c->cond.offset;
    for (int i = 0; i < 4; i++) c->conf.qf[i] = (float)c->cond.qf[i];
    for (int i = 0; i < 9; i++) c->conf.rft[i] = (float)c->cond.rft[i];
    c->conf.weight = (float)c->cond.weight;
    return 0;
}

int cprrtc_prepare(void* p, int width) {
    Ctx* c = C(p);
    if (!c) return fail(CPRRTC_EARG, "NULL context");
    if (int rc = set_device(c)) return rc;
    Module* m;
    return cur_module(c, width, 0, &m);
}

int64_t cprrtc_launch_count(void* p) { return p ? C(p)->launches : 0; }

int cprrtc_last_timing(void* p, double* total_ms, double* plan_ms) {
    Ctx* c = C(p);
    if (!c) return fail(CPRRTC_EARG, "NULL context");
    if (c->timing_pending && c->plan_lean) {   // no events in the lean graph: the kernel's own clock
        c->last_total_ms = c->last_kernel_total_ms;
        c->last_plan_ms = c->last_query_ms;
        c->timing_pending = false;
    }
    if (c->timing_pending) {
        float t_all = 0, t_plan = 0;
        if (int rc = set_device(c)) return rc;
        cudaEventSynchronize(c->ev[3]);   // plan_collect returns before the graph's results event
        cudaEventElapsedTime(&t_all, c->ev[0], c->ev[3]);
        // without events around the planner (the PDL graph) its time is the
        // longest query's device time (init -> solved / last team out, globaltimer)
        if (c->plan_ev) cudaEventElapsedTime(&t_plan, c->ev[1], c->ev[2]);
        else t_plan = (float)c->last_query_ms;
        c->last_total_ms = t_all;
        c->last_plan_ms = t_plan;
        c->timing_pending = false;
    }
    if (total_ms) *total_ms = c->last_total_ms;
    if (plan_ms) *plan_ms = c->last_plan_ms;
    return 0;
}

int cprrtc_flush_l2(void* p, size_t bytes) {
    Ctx* c = C(p);
    if (!c) return fail(CPRRTC_EARG, "NULL context");
    if (int rc = set_device(c)) return rc;
    if (int rc = c->scratch[8].ensure(bytes)) return rc;
    CUDA_TRY(cudaMemsetAsync(c->scratch[8].p, (int)(c->launches & 0xff), bytes, c->stream));
    return sync(c);
}

int cprrtc_fk(void* p, int B, const double* q, int fp64, double* frames, double* axes, double* origins, double* ee,
              double* spheres) {
    Ctx* c = C(p);
    if (!c || B < 0 || (B && !q)) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    const int n = c->n, S = c->S;
    int rc = upload(c, c->scratch[0], q, (size_t)B * n);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * n * 12 * 8);
    rc = rc ? rc : c->scratch[2].ensure((size_t)B * n * 3 * 8);
    rc = rc ? rc : c->scratch[3].ensure((size_t)B * n * 3 * 8);
    rc = rc ? rc : c->scratch[4].ensure((size_t)B * 7 * 8);
    rc = rc ? rc : c->scratch[5].ensure((size_t)B * (S ? S : 1) * 4 * 8);
    if (rc) return rc;
    const double* dq = c->scratch[0].as<double>();
    double* df = frames ? c->scratch[1].as<double>() : nullptr;
    double* da = (axes || origins) ? c->scratch[2].as<double>() : nullptr;
    double* dor = (axes || origins) ? c->scratch[3].as<double>() : nullptr;
    double* de = ee ? c->scratch[4].as<double>() : nullptr;
    double* ds = spheres ? c->scratch[5].as<double>() : nullptr;
    void* args[] = {&B, &fp64, &dq, &df, &da, &dor, &de, &ds};
    if (int rc2 = launch(c, m, "cp_fk_kernel", (B + 127) / 128, 1, 128, 0, args)) return rc2;
    if (frames) download(c, frames, c->scratch[1], (size_t)B * n * 12);
    if (axes) download(c, axes, c->scratch[2], (size_t)B * n * 3);
    if (origins) download(c, origins, c->scratch[3], (size_t)B * n * 3);
    if (ee) download(c, ee, c->scratch[4], (size_t)B * 7);
    if (spheres) download(c, spheres, c->scratch[5], (size_t)B * S * 4);
    return sync(c);
}

int cprrtc_task_err_jac(void* p, int B, const double* q, int fp64, double* e, double* J) {
    Ctx* c = C(p);
    if (!c || B < 0 || (B && (!q || !e || !J))) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    const int M = (c->kind == 0 ? 1 : 2) + (c->orient ? 3 : 0);
    int rc = upload(c, c->scratch[0], q, (size_t)B * c->n);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * M * 8);
    rc = rc ? rc : c->scratch[2].ensure((size_t)B * M * c->n * 8);
    if (rc) return rc;
    const double* dq = c->scratch[0].as<double>();
    double* de = c->scratch[1].as<double>();
    double* dJ = c->scratch[2].as<double>();
    void* args[] = {&B, &fp64, &c->conf, &c->cond, &dq, &de, &dJ};
    if (int rc2 = launch(c, m, "cp_tej_kernel", (B + 127) / 128, 1, 128, 0, args)) return rc2;
    download(c, e, c->scratch[1], (size_t)B * M);
    download(c, J, c->scratch[2], (size_t)B * M * c->n);
    return sync(c);
}

int cprrtc_task_error_at(void* p, int B, const double* pose7, double* e) {
    Ctx* c = C(p);
    if (!c || B < 0 || (B && (!pose7 || !e))) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    const int M = (c->kind == 0 ? 1 : 2) + (c->orient ? 3 : 0);
    int rc = upload(c, c->scratch[0], pose7, (size_t)B * 7);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * M * 8);
    if (rc) return rc;
    const double* dp = c->scratch[0].as<double>();
    double* de = c->scratch[1].as<double>();
    void* args[] = {&B, &c->cond, &dp, &de};
    if (int rc2 = launch(c, m, "cp_err_at_kernel", (B + 127) / 128, 1, 128, 0, args)) return rc2;
    download(c, e, c->scratch[1], (size_t)B * M);
    return sync(c);
}

int cprrtc_project_config(void* p, int B, double* q_io, double tau, double lam, int max_iters, int32_t* ok) {
    Ctx* c = C(p);
    if (!c || B < 0 || (B && (!q_io || !ok))) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    int rc = upload(c, c->scratch[0], q_io, (size_t)B * c->n);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * 4);
    if (rc) return rc;
    double* dq = c->scratch[0].as<double>();
    int* dok = c->scratch[1].as<int>();
    void* args[] = {&B, &c->cond, &tau, &lam, &max_iters, &dq, &dok};
    if (int rc2 = launch(c, m, "cp_project_config_kernel", (B + 63) / 64, 1, 64, 0, args)) return rc2;
    download(c, q_io, c->scratch[0], (size_t)B * c->n);
    download(c, ok, c->scratch[1], (size_t)B);
    return sync(c);
}

static SetupArgs setup_args(Ctx* c, double tau) {
    SetupArgs S;
    std::memset(&S, 0, sizeof S);
    S.con = c->cond;
    S.tau_task = tau;
    S.box_min = c->sc_bmin.as<double>();
    S.box_max = c->sc_bmax.as<double>();
    S.sph_c = c->sc_sc.as<double>();
    S.sph_r = c->sc_sr.as<double>();
    S.nb = c->nb;
    S.ne = c->ne;
    return S;
}

int cprrtc_check_config(void* p, int B, const double* q, double tau, int32_t* code) {
    Ctx* c = C(p);
    if (!c || B < 0 || (B && (!q || !code))) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    int rc = upload(c, c->scratch[0], q, (size_t)B * c->n);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * 4);
    if (rc) return rc;
    SetupArgs S = setup_args(c, tau);
    const double* dq = c->scratch[0].as<double>();
    int* dc = c->scratch[1].as<int>();
    void* args[] = {&B, &S, &dq, &dc};
    if (int rc2 = launch(c, m, "cp_check_config_kernel", (B + 3) / 4, 1, 128, 0, args)) return rc2;
    download(c, code, c->scratch[1], (size_t)B);
    return sync(c);
}

static int validate_impl(void* p, int B, int W, const double* wps, int flag_on, double margin, int cull,
                         int32_t* valid, int32_t* first_bad, int64_t* performed, int64_t* possible,
                         int64_t* gpu_checks) {
    Ctx* c = C(p);
    if (!c || B < 0 || W < 1 || (B && (!wps || !valid || !first_bad || !performed)))
        return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (W > 32) return fail(CPRRTC_ELIMIT, "at most 32 waypoints per motion in this build");
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, W <= 16 ? 16 : 32, c->kind, c->orient, 1, &m)) return rc;
    int rc = upload(c, c->scratch[0], wps, (size_t)B * W * c->n);
    rc = rc ? rc : c->scratch[1].ensure((size_t)B * 4);
    rc = rc ? rc : c->scratch[2].ensure((size_t)B * 4);
    rc = rc ? rc : c->scratch[3].ensure((size_t)B * 8);
    rc = rc ? rc : c->scratch[4].ensure((size_t)B * 8);
    if (rc) return rc;
    SceneSm sc = scene_args(c, cull);
    const double* dw = c->scratch[0].as<double>();
    int* dv = c->scratch[1].as<int>();
    int* df = c->scratch[2].as<int>();
    int64_t* dp = c->scratch[3].as<int64_t>();
    int64_t* dg = c->scratch[4].as<int64_t>();
    float mg = (float)margin;
    void* args[] = {&B, &W, &flag_on, &mg, &sc, &dw, &dv, &df, &dp, &dg};
    const int tpc = kThreads / m->G;
    int grid = (B + tpc - 1) / tpc;
    if (grid > 64 * c->sms) grid = 64 * c->sms;
    CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
    if (int rc2 = launch(c, m, cull ? "cp_validate_cull_kernel" : "cp_validate_kernel", grid, 1, kThreads,
                         team_smem(c, m, true), args))
        return rc2;
    CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
    download(c, valid, c->scratch[1], (size_t)B);
    download(c, first_bad, c->scratch[2], (size_t)B);
    download(c, performed, c->scratch[3], (size_t)B);
    if (gpu_checks) download(c, gpu_checks, c->scratch[4], (size_t)B);
    if (int rc3 = sync(c)) return rc3;
    {
        float t = 0;
        cudaEventElapsedTime(&t, c->ev[1], c->ev[2]);
        c->last_plan_ms = t;
        c->last_total_ms = t;
        c->timing_pending = false;
    }
    if (possible) {
        const int64_t per = (int64_t)c->S * (c->nb + c->ne) + c->P;
        for (int i = 0; i < B; i++) possible[i] = per * W;
    }
    return 0;
}

int cprrtc_validate(void* p, int B, int W, const double* wps, int flag_on, double margin, int32_t* valid,
                    int32_t* first_bad, int64_t* performed, int64_t* possible, int64_t* gpu_checks) {
    return validate_impl(p, B, W, wps, flag_on, margin, 0, valid, first_bad, performed, possible, gpu_checks);
}

int cprrtc_validate_broadphase(void* p, int B, int W, const double* wps, int flag_on, double margin,
                               int32_t* valid, int32_t* first_bad, int64_t* performed, int64_t* possible,
                               int64_t* gpu_checks) {
    return validate_impl(p, B, W, wps, flag_on, margin, 1, valid, first_bad, performed, possible, gpu_checks);
}

int cprrtc_project(void* p, int B, int W, const double* wps, const double* tau_sm, double tau_task, double alpha,
                   double lam, int max_iters, int mode, double* xi, int32_t* ok, int32_t* iters, int32_t* prog,
                   double* trace, int32_t* trace_prog) {
    Ctx* c = C(p);
    if (!c || B < 0 || W < 2 || max_iters < 1 || mode < 0 || mode > 2 ||
        (B && (!wps || !xi || !ok || !iters || !prog)))
        return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = cur_module(c, W, 1, &m)) return rc;
    const size_t nw = (size_t)B * W * c->n;
    int rc = upload(c, c->scratch[0], wps, nw);
    rc = rc ? rc : c->scratch[1].ensure(nw * 8);
    rc = rc ? rc : c->scratch[2].ensure((size_t)B * 12);
    if (rc) return rc;
    std::vector<float> tsm;
    if (tau_sm) {
        tsm.resize(B);
        for (int i = 0; i < B; i++) tsm[i] = (float)tau_sm[i];
        if ((rc = upload(c, c->scratch[3], tsm.data(), (size_t)B))) return rc;
    }
    float* dtrace = nullptr;
    int* dtp = nullptr;
    if (trace) {
        rc = c->scratch[4].ensure((size_t)B * max_iters * W * c->n * 4);
        rc = rc ? rc : c->scratch[5].ensure((size_t)B * max_iters * 4);
        if (rc) return rc;
        CUDA_TRY(cudaMemsetAsync(c->scratch[5].p, 0xff, (size_t)B * max_iters * 4, c->stream));
        dtrace = c->scratch[4].as<float>();
        dtp = c->scratch[5].as<int>();
    }
    ProjArgs pa{};
    pa.alpha = (float)alpha;
    pa.lam = (float)lam;
    pa.tau_task = (float)tau_task;
    pa.tau_task_dev = tau_dev(tau_task);
    pa.tau_sm_fixed = 0.f;
    pa.max_iters = max_iters;
    pa.mode = mode;
    const double* dw = c->scratch[0].as<double>();
    double* dxi = c->scratch[1].as<double>();
    int* dok = c->scratch[2].as<int>();
    int* dit = dok + B;
    int* dpr = dok + 2 * B;
    const float* dts = tau_sm ? c->scratch[3].as<float>() : nullptr;
    void* args[] = {&B, &W, &c->conf, &pa, &dts, &dw, &dxi, &dok, &dit, &dpr, &dtrace, &dtp};
    const int tpc = kThreads / m->G;
    int grid = (B + tpc - 1) / tpc;
    if (grid > 64 * c->sms) grid = 64 * c->sms;
    if (int rc2 = upload_conf(c, m)) return rc2;
    if (int rc2 = launch(c, m, "cp_project_kernel", grid, 1, kThreads, team_smem(c, m, false), args)) return rc2;
    download(c, xi, c->scratch[1], nw);
    std::vector<int> tmp((size_t)3 * B);
    download(c, tmp.data(), c->scratch[2], (size_t)3 * B);
    std::vector<float> tr;
    if (trace) {
        tr.resize((size_t)B * max_iters * W * c->n);
        download(c, tr.data(), c->scratch[4], tr.size());
        download(c, trace_prog, c->scratch[5], (size_t)B * max_iters);
    }
    if (int rc3 = sync(c)) return rc3;
    for (int i = 0; i < B; i++) {
        ok[i] = tmp[i];
        iters[i] = tmp[B + i];
        prog[i] = tmp[2 * B + i];
    }
    if (trace)
        for (size_t i = 0; i < tr.size(); i++) trace[i] = tr[i];
    return 0;
}

int cprrtc_nearest_trees(void* p, int N, int n_trees, const float* soa_dev_or_null, const double* nodes, int Q,
                         const double* queries, int32_t* idx);

int cprrtc_nearest(void* p, int N, const double* nodes, int Q, const double* queries, int32_t* idx) {
    return cprrtc_nearest_trees(p, N, 1, nullptr, nodes, Q, queries, idx);
}

// Q queries; query i scans tree (i % n_trees), each of N nodes.  nodes:
// (n_trees, N, n) row-major host array (converted to the SoA device layout).
int cprrtc_nearest_trees(void* p, int N, int n_trees, const float* unused, const double* nodes, int Q,
                         const double* queries, int32_t* idx) {
    (void)unused;
    Ctx* c = C(p);
    if (!c || N < 1 || n_trees < 1 || Q < 0 || !nodes || (Q && (!queries || !idx)))
        return fail(CPRRTC_EARG, "bad argument");
    if (Q == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    const int n = c->n;
    const int cap = (N + 127) / 128 * 128;
    std::vector<float> soa((size_t)n_trees * n * cap, NAN);
    for (int t = 0; t < n_trees; t++)
        for (int i = 0; i < N; i++)
            for (int k = 0; k < n; k++)
                soa[((size_t)t * n + k) * cap + i] = (float)nodes[((size_t)t * N + i) * n + k];
    std::vector<float> qf((size_t)Q * n);
    for (size_t i = 0; i < qf.size(); i++) qf[i] = (float)queries[i];
    int rc = upload(c, c->scratch[0], soa.data(), soa.size());
    rc = rc ? rc : upload(c, c->scratch[1], qf.data(), qf.size());
    rc = rc ? rc : c->scratch[2].ensure((size_t)Q * 4);
    if (rc) return rc;
    const float* dn = c->scratch[0].as<float>();
    const float* dq = c->scratch[1].as<float>();
    int* di = c->scratch[2].as<int>();
    void* args[] = {&N, (void*)&cap, &n_trees, &dn, &Q, &dq, &di};
    const int tpc = kThreads / m->G;
    int grid = (Q + tpc - 1) / tpc;
    if (grid > 64 * c->sms) grid = 64 * c->sms;
    CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
    if (int rc2 = launch(c, m, "cp_nearest_kernel", grid, 1, kThreads, 0, args)) return rc2;
    CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
    download(c, idx, c->scratch[2], (size_t)Q);
    if (int rc3 = sync(c)) return rc3;
    float t = 0;
    cudaEventElapsedTime(&t, c->ev[1], c->ev[2]);
    c->last_plan_ms = c->last_total_ms = t;
    c->timing_pending = false;
    return 0;
}

int cprrtc_halton(void* p, int count, int64_t first_index, int64_t seed_offset, const double* lo, const double* hi,
                  double* out) {
    Ctx* c = C(p);
    if (!c || count < 0 || (count && !out) || first_index < 0 || seed_offset < 0)
        return fail(CPRRTC_EARG, "bad argument");
    if (count == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = get_module(c, 16, c->kind, c->orient, 1, &m)) return rc;
    if (int rc = c->scratch[0].ensure((size_t)count * c->n * 8)) return rc;
    if (int rc = upload(c, c->scratch[1], lo ? lo : c->lo.data(), (size_t)c->n)) return rc;
    if (int rc = upload(c, c->scratch[2], hi ? hi : c->hi.data(), (size_t)c->n)) return rc;
    double* d = c->scratch[0].as<double>();
    const double* dlo = c->scratch[1].as<double>();
    const double* dhi = c->scratch[2].as<double>();
    long long fi = first_index, so = seed_offset;
    void* args[] = {&count, &fi, &so, &dlo, &dhi, &d};
    if (int rc2 = launch(c, m, "cp_halton_kernel", (count + 127) / 128, 1, 128, 0, args)) return rc2;
    download(c, out, c->scratch[0], (size_t)count * c->n);
    return sync(c);
}

static int ensure_plan_buffers(Ctx* c, int nq, int cap, int path_cap) {
    const int n = c->n;
    if (nq > c->nq_alloc || cap != c->cap_alloc) {
        size_t tree_bytes = (size_t)nq * 2 * n * cap * sizeof(float);
        int rc = c->trees.ensure(tree_bytes);
        rc = rc ? rc : c->parents.ensure((size_t)nq * 2 * cap * sizeof(int));
        rc = rc ? rc : c->qs.ensure((size_t)nq * sizeof(QueryState));
        if (rc) return rc;
        for (auto& g : c->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        c->graphs.clear();
        CUDA_TRY(cudaMemsetAsync(c->trees.p, 0xff, tree_bytes, c->stream));   // NaN = unpublished
        CUDA_TRY(cudaMemsetAsync(c->parents.p, 0xff, (size_t)nq * 2 * cap * sizeof(int), c->stream));   // -1
        CUDA_TRY(cudaMemsetAsync(c->qs.p, 0, (size_t)nq * sizeof(QueryState), c->stream));
        c->nq_alloc = nq;
        c->cap_alloc = cap;
    }
    int rc = c->counters.ensure(64);
    {   // inputs (starts | goals | seeds) in one block; a move invalidates the graphs
        void* before = c->d_starts.p;
        rc = rc ? rc : c->d_starts.ensure((size_t)nq * (2 * n + 1) * 8 + 8);   // + the call's sequence number
        void* hbefore = c->h_in.h;
        rc = rc ? rc : c->h_in.ensure((size_t)nq * (2 * n + 1) * 8 + 8);
        void* obefore = c->h_out.h;
        rc = rc ? rc : c->h_out.ensure((size_t)nq * sizeof(QueryOut));
        void* pbefore = c->h_paths.h;
        rc = rc ? rc : c->h_paths.ensure((size_t)nq * path_cap * n * sizeof(float));
        void* sbefore = c->h_src.h;
        rc = rc ? rc : c->h_src.ensure((size_t)nq * path_cap * sizeof(int));
        void* cbefore = c->chain.p;
        rc = rc ? rc : c->chain.ensure((size_t)nq * path_cap * sizeof(int));
        if (before != c->d_starts.p || hbefore != c->h_in.h || obefore != c->h_out.h || pbefore != c->h_paths.h ||
            sbefore != c->h_src.h || cbefore != c->chain.p) {
            for (auto& g : c->graphs)
                if (g.exec) cudaGraphExecDestroy(g.exec);
            c->graphs.clear();
        }
    }

    c->path_cap = path_cap;
    return rc;
}

static PlanArgs make_plan_args(Ctx* c, const cprrtc_params* prm, int B, int cap, double tau) {
    PlanArgs A;
    std::memset(&A, 0, sizeof A);   // padding too: graphs are keyed by the raw bytes
    A.qs = c->qs.as<QueryState>();
    A.trees = c->trees.as<float>();
    A.parents = c->parents.as<int>();
    A.cap = cap;
    A.nq = B;
    A.queue_head = c->counters.as<int>();
    A.team_counter = c->counters.as<int>() + 1;
    // broad phase: explicit, or (-1) whenever the scene has obstacles (r1 A/B
    // on upright Panda, 6 primitives: 0.367 vs 0.395 ms median lockstep)
    A.scene_g = scene_args(c, prm->cc_broadphase < 0 ? (c->nb + c->ne > 0) : prm->cc_broadphase != 0);
    A.con = c->conf;
    A.pa.alpha = (float)prm->alpha;
    A.pa.lam = (float)prm->lam;
    A.pa.tau_task = (float)tau;
    A.pa.tau_task_dev = tau_dev(tau);
    A.pa.tau_sm_fixed = prm->tau_sm > 0 ? (float)prm->tau_sm : 0.f;
    A.pa.max_iters = prm->proj_max_iters;
    A.pa.mode = prm->projection_mode;
    A.W = prm->width;
    A.step = (float)prm->step_size;
    A.tol = (float)(prm->connect_tolerance > 0 ? prm->connect_tolerance : prm->step_size / 10.0);
    A.margin = (float)prm->cc_margin;
    A.flag_on = prm->flag_on;
    A.max_iterations = prm->max_iterations;
    A.max_connect = prm->max_connect_segments;
    // 0: no budget (deterministic); -1: already expired (time_budget_ms <= 0)
    A.budget_ns = prm->deterministic ? 0 : (prm->time_budget_ms <= 0 ? -1 : (i64)(prm->time_budget_ms * 1e6));
    return A;
}

static int check_params(const cprrtc_params* prm) {
    if (prm->step_size <= 0 || prm->width < 2 || prm->max_iterations < 1 || prm->alpha <= 0 || prm->lam < 0 ||
        prm->proj_max_iters < 1 || prm->projection_mode < 0 || prm->projection_mode > 2)
        return fail(CPRRTC_EARG, "invalid planner parameters");
    return 0;
}

// First-solution race of one query across contexts (devices): every racer
// polls its own flag word; the winner stores 1 into every racer's word (peer
// stores over NVLink, or one shared mapped host word without peer access).
struct RaceLink {
    int* own;
    int* peers[CPRRTC_MAX_RACE];
    int n;
};

// Stage inputs and launch the per-call sequence (H2D, setup, plan, extract)
// on the context's stream; plan_collect waits and reads the results.
static int plan_collect(Ctx* c, int B, cprrtc_result* results, double* paths, int32_t* sources);

// A solved path's roots are the exact FP64 endpoints (the tree roots hold
// their FP32 roundings on the device)
static void exact_roots(const Ctx* c, int B, const double* starts, const double* goals, const cprrtc_result* results,
                        double* paths) {
    if (!paths) return;
    const int n = c->n;
    for (int i = 0; i < B; i++) {
        const int L = results[i].path_len;
        if (L < 2) continue;
        double* row = paths + (size_t)i * c->path_cap * n;
        std::memcpy(row, starts + (size_t)i * n, (size_t)n * sizeof(double));
        std::memcpy(row + (size_t)(L - 1) * n, goals + (size_t)i * n, (size_t)n * sizeof(double));
    }
}

// Developer knob: CPRRTC_HOST_PROFILE=1 prints, at exit, the medians of the
// host-side phases of cprrtc_plan (us): launch preparation, cudaGraphLaunch,
// the wait for the results event, the result copy.
namespace {
struct HostProfile {
    std::vector<double> v[4];
    ~HostProfile() {
        if (v[0].empty()) return;
        const char* names[4] = {"prepare", "graph launch", "wait", "collect"};
        std::fprintf(stderr, "[cprrtc host profile] %zu calls, medians (us):", v[0].size());
        for (int k = 0; k < 4; k++) {
            std::vector<double> x = v[k];
            std::nth_element(x.begin(), x.begin() + x.size() / 2, x.end());
            std::fprintf(stderr, " %s %.2f", names[k], x[x.size() / 2]);
        }
        std::fprintf(stderr, "\n");
    }
};
HostProfile g_hprof;
double g_hp_launch_us = 0.0;   // cudaGraphLaunch time of the last plan_launch
const bool g_hp_on = getenv("CPRRTC_HOST_PROFILE") && atoi(getenv("CPRRTC_HOST_PROFILE")) != 0;
}  // namespace

static int plan_launch(Ctx* c, const cprrtc_params* prm, int B, const double* starts, const double* goals,
                       const int64_t* seeds, const RaceLink* race) {
    if (c->inflight) return fail(CPRRTC_EARG, "the context has a submitted batch not yet waited for");
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = cur_module(c, prm->width, 0, &m)) return rc;
    const int n = c->n;
    // tree capacity: every sample adds at most 1 + max_connect_segments nodes
    long long want = prm->tree_capacity > 0 ? prm->tree_capacity
                                            : (long long)prm->max_iterations * (1 + prm->max_connect_segments) / 2 + 256;
    long long budget_nodes = (1ll << 30) / ((long long)B * 2 * n * 4 + 1) * 4;   // ~4 GiB of trees
    if (prm->tree_capacity <= 0 && want > budget_nodes) want = budget_nodes;
    if (want > (1 << 26)) want = 1 << 26;
    int cap = (int)((want + 127) / 128 * 128);
    if (cap < 128) cap = 128;
    const int path_cap = prm->path_capacity > 0 ? prm->path_capacity : 1024;
    if (int rc = ensure_plan_buffers(c, B, cap, path_cap)) return rc;
    // inputs: one pinned staging block (starts | goals | seeds) -> one H2D copy
    double* hin = c->h_in.host<double>();
    std::memcpy(hin, starts, (size_t)B * n * 8);
    std::memcpy(hin + (size_t)B * n, goals, (size_t)B * n * 8);
    long long* hseed = reinterpret_cast<long long*>(hin + (size_t)2 * B * n);
    for (int i = 0; i < B; i++) hseed[i] = seeds ? seeds[i] : 0;
    hseed[B] = (long long)++c->plan_seq;   // the completion words carry it back (plan_collect)
    const size_t in_bytes = (size_t)B * (2 * n + 1) * 8 + 8;
    const double tau = prm->tau_task > 0 ? prm->tau_task : c->tau_task;
    // setup (FP64 endpoint checks, NaN refill of last run's slots, roots,
    // counters) -- planner.py:416-445
    SetupArgs S = setup_args(c, tau);
    S.qs = c->qs.as<QueryState>();
    S.starts = c->d_starts.as<double>();
    S.goals = S.starts + (size_t)B * n;
    S.seeds = reinterpret_cast<const i64*>(S.starts + (size_t)2 * B * n);
    S.trees = c->trees.as<float>();
    S.parents = c->parents.as<int>();
    S.cap = cap;
    S.counters = c->counters.as<int>();
    // the persistent planner
    PlanArgs A = make_plan_args(c, prm, B, cap, tau);
    A.out = c->h_out.dev<QueryOut>();
    A.paths = c->h_paths.dev<float>();
    A.sources = c->h_src.dev<int>();
    A.chain = c->chain.as<int>();
    A.path_cap = path_cap;
    A.seeds = S.seeds;
    S.out = A.out;
    if (race) {
        A.race_flag = race->own;
        A.n_race = race->n;
        for (int k = 0; k < race->n; k++) A.race_peers[k] = race->peers[k];
    }
    if (!m->plan_occ) {
        int occ = 0;
        drv().occupancy(&occ, m->fn["cp_plan_kernel"], kThreads, team_smem(c, m, true));
        m->plan_occ = occ > 0 ? occ : 1;
    }
    // single queries run one team per warp (latency); batches pack two (G=16)
    const bool solo = B == 1 && m->G == 16 && !(prm->teams < 0);
    // two-warp teams (P projects, C certifies one motion behind) for single
    // queries; CPRRTC_PAIR=0 restores one-warp teams.  r1 sweep (upright Panda,
    // one box): one-warp 512 teams 0.202 ms median / p90 0.383; pairs 192 /
    // 256 / 320 / 384 -> 0.178 / 0.177 / 0.185 / 0.186 ms, p90 0.334-0.343
    // (r1 A/B on the 999-box shelf: pairs also win for unconstrained queries,
    // arm8 0.28 -> 0.23 ms, arm7 equal)
    // (r1 re-sweep after the fast start, tools/team_sweep.sh: 160-222 pairs
    // ~2 % under 256 on upright Panda, but the shelf and configs[3] medians
    // 4-5 % over; 256 kept.  r2 re-sweep on the r2 code, every config,
    // tools/team_sweep_all.py: 128 / 148 / 160 / 192 / 256 pairs -> upright
    // 0.144 / 0.142 / 0.145 / 0.144 / 0.148-0.151 ms, 999-box shelf 0.199 /
    // 0.209 / 0.187 / 0.180 / 0.190, configs[3] 0.200 / 0.207 / 0.205 / 0.202 /
    // 0.205-0.208, configs[0] equal: 192 pairs)
    static const bool pair_off = getenv("CPRRTC_PAIR") && atoi(getenv("CPRRTC_PAIR")) == 0;
    const bool pair = solo && !pair_off;
    const int tpw = solo ? 1 : 32 / m->G;         // teams per warp
    const int max_tpc = solo ? kThreads / 32 : kThreads / m->G;   // teams per full CTA
    const int resident = m->plan_occ * c->sms * max_tpc;
    // concurrency: the requested team count, else (single query) 192 pair
    // teams / 512 one-warp teams, or (batches) B + B/8 teams but at least half
    // the resident ones -- r2 sweep, 1024-query batches (tools/batch_teams.py):
    // 592 / 740 / 1036 / 1184 / 1480 / 2368 (every resident) teams -> 0.98 /
    // 0.99 / 1.08 / 1.13 / 1.09 / 0.94 M queries/s: past ~one team per query the
    // extra teams mostly duplicate work the first solution throws away; never
    // more than a quarter of the sample budget so that at least ~4 waves of
    // extensions build on each other (samples are the reference's iterations)
    long long want_teams = prm->teams > 0 ? prm->teams
                           : (B == 1 ? (pair ? 192 : 512) : std::max((long long)B + B / 8, (long long)resident / 2));
    long long budget_teams = (long long)B * prm->max_iterations / 4;
    if (budget_teams < tpw) budget_teams = tpw;
    if (want_teams > budget_teams) want_teams = budget_teams;
    if (want_teams > resident) want_teams = resident;
    // spread the teams over every SM first (latency of a team is set by how
    // many warps share its SM), then fill CTAs up to 256 threads
    if (pair) want_teams *= 2;                    // warps: one P and one C per team
    long long per_cta = (want_teams + c->sms - 1) / c->sms;
    per_cta = (per_cta + tpw - 1) / tpw * tpw;
    if (pair) per_cta = (per_cta + 1) / 2 * 2;    // whole pairs per CTA
    if (per_cta > max_tpc) per_cta = max_tpc;
    const int block = (int)(per_cta * 32 / tpw);
    int grid = (int)((want_teams + per_cta - 1) / per_cta);
    if (grid < 1) grid = 1;
    const size_t smem = scene_smem(c, A.scene_g.cull) + (size_t)(block / m->G) * m->ws_bytes;
    A.solo = solo ? 1 : 0;
    A.pair = pair ? 1 : 0;
    // the lean single-query graph: H2D -> init -> planner -> reset, no event
    // records and no endpoint-check kernel (the first two teams' certifier
    // warps check the endpoints; the host waits on completion words).  r2
    // same-box A/B, upright Panda: e2e median -5 to -9 us (each graph node
    // costs launch and scheduling latency, and the FP64 check kernel shared
    // the SMs with the planner's first wave).  Races keep the events
    // (cprrtc_elapsed_ms), and so does CPRRTC_PDL=0.
    static const bool pdl_on = !(getenv("CPRRTC_PDL") && atoi(getenv("CPRRTC_PDL")) == 0);
    const bool lean = pair && !race && pdl_on;
    A.chk_in_kernel = lean ? 1 : 0;
    if (pair) A.chk = S;   // (the pair planner also reads the roots' FP64 inputs through it)
    if (int rc = upload_conf(c, m)) return rc;
    // the per-call sequence as one CUDA graph, replayed while shapes and
    // arguments repeat (inputs change only inside the pinned staging block)
    Ctx::PlanGraph* G = nullptr;
    for (auto& g : c->graphs)
        if (g.m == m && g.B == B && g.grid == grid && g.block == block && g.smem == smem &&
            g.path_cap == path_cap && !std::memcmp(&g.A, &A, sizeof A) && !std::memcmp(&g.S, &S, sizeof S)) {
            G = &g;
            break;
        }
    if (!G) {
        if (c->graphs.size() >= 8) {
            cudaGraphExecDestroy(c->graphs.front().exec);
            c->graphs.erase(c->graphs.begin());
        }
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const int64_t launches0 = c->launches;
        int rc = 0;
        cudaMemcpyAsync(c->d_starts.p, hin, in_bytes, cudaMemcpyHostToDevice, c->stream);
        if (!lean) {
            cudaEventRecordWithFlags(c->ev[0], c->stream, cudaEventRecordExternal);   // device-resident inputs from here on
            // FP64 endpoint checks on a concurrent branch (they only veto a query;
            // the init kernel leaves their stop / setup words alone)
            cudaEventRecord(c->fork, c->stream);
            cudaStreamWaitEvent(c->stream2, c->fork, 0);
            {
                void* args[] = {&S};
                rc = rc ? rc : launch(c, m, "cp_check_kernel", B, 1, 64, 0, args, c->stream2);
            }
            cudaEventRecord(c->join, c->stream2);
        }
        // the planner is a programmatic dependent of init (its scene staging
        // overlaps init) with no event nodes around it: r1 A/B on one box,
        // upright Panda median 0.158 -> 0.148 ms (events 5 %, PDL 2 %);
        // CPRRTC_PDL=0 restores a plain launch bracketed by ev[1] / ev[2]
        static const bool pdl = !(getenv("CPRRTC_PDL") && atoi(getenv("CPRRTC_PDL")) == 0);
        const bool noev = pdl;
        {   // query state + roots
            void* args[] = {&S};
            rc = rc ? rc : launch(c, m, "cp_init_kernel", B, 1, 32, 0, args);
        }
        if (!noev) cudaEventRecordWithFlags(c->ev[1], c->stream, cudaEventRecordExternal);
        {   // the persistent planner; the last team out of each query extracts its result
            void* args[] = {&A};
            rc = rc ? rc : (pdl ? launch_pdl(c, m, "cp_plan_kernel", grid, block, smem, args)
                                : launch(c, m, "cp_plan_kernel", grid, 1, block, smem, args));
        }
        if (!noev) cudaEventRecordWithFlags(c->ev[2], c->stream, cudaEventRecordExternal);
        c->plan_ev = !noev;
        if (!lean) {
            cudaStreamWaitEvent(c->stream, c->join, 0);
            cudaEventRecordWithFlags(c->ev[3], c->stream, cudaEventRecordExternal);   // results complete
        }
        {   // NaN-refill this run's node slots for the next run (after ev[3]: the
            // host waits on ev[3] only, so this overlaps the host's result handling)
            QueryState* qs = c->qs.as<QueryState>();
            float* tr = c->trees.as<float>();
            int* pa = c->parents.as<int>();
            int capv = cap, nq = B;
            void* args[] = {&qs, &tr, &pa, &capv, &nq};
            rc = rc ? rc : launch(c, m, "cp_reset_kernel", 8, (unsigned)std::min(2 * B, 65535), 256, 0, args);
        }
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
        c->launches = launches0;
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        Ctx::PlanGraph g;
        g.A = A;
        g.S = S;
        g.B = B;
        g.grid = grid;
        g.block = block;
        g.smem = smem;
        g.path_cap = path_cap;
        g.m = m;
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        c->graphs.push_back(g);
        G = &c->graphs.back();
    }
    {
        const auto tl = g_hp_on ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point();
        CUDA_TRY(cudaGraphLaunch(G->exec, c->stream));
        if (g_hp_on)
            g_hp_launch_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tl).count();
    }
    c->launches += lean ? 3 : 4;   // init, (check,) plan, reset
    c->plan_lean = lean;
    c->last_args = A;
    c->last_mod = m;
    c->last_nq = B;
    return 0;
}

// Wait for a launch's results.  A single query's completion words (written
// in mapped memory by its finalizer and its endpoint check, behind
// system-scope fences) carry the launch's sequence number -- the host sees
// them a PCIe write after the last team leaves, without waiting for the
// planner grid to retire and the graph's results event to fire (r2: e2e
// median -8 %).  The event is still queried every few thousand polls: a
// failed launch, or one that ended without writing a word, ends the wait
// there.  Batches wait for the event: there the system-scope fences, one per
// query and per solved path, cost more than they save (r2: 1024-query batch
// kernel 0.84 -> 1.21 ms with them).
static int wait_results(Ctx* c, int B) {
    if (B != 1) {
        const cudaError_t e = cudaEventSynchronize(c->ev[3]);
        if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("kernel failed: ") + cudaGetErrorString(e));
        return 0;
    }
    const volatile QueryOut* out = c->h_out.host<QueryOut>();
    const unsigned seq = c->plan_seq;
    for (unsigned spin = 1;; spin++) {
        bool all = true;
        for (int i = 0; i < B && all; i++) all = out[i].done_seq == seq && out[i].chk_seq == seq;
        if (all) break;
        if ((spin & 4095) == 0) {
            const cudaError_t e = c->plan_lean ? cudaStreamQuery(c->stream) : cudaEventQuery(c->ev[3]);
            if (e == cudaSuccess) {
                // the launch is complete, so its mapped-memory stores are
                // visible: words still from an earlier call mean a result
                // that was never written -- never hand that back as this call's
                for (int i = 0; i < B; i++)
                    if (out[i].done_seq != seq || out[i].chk_seq != seq)
                        return fail(CPRRTC_ECUDA, "launch completed without writing its results");
                break;
            }
            if (e != cudaErrorNotReady)
                return fail(CPRRTC_ECUDA, std::string("kernel failed: ") + cudaGetErrorString(e));
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return 0;
}

static int plan_collect(Ctx* c, int B, cprrtc_result* results, double* paths, int32_t* sources) {
    if (int rc = set_device(c)) return rc;
    // results are complete when the completion words say so; the planner's
    // last warps, the results event and the tree refill behind it may still run
    if (int rc = wait_results(c, B)) return rc;
    const int n = c->n;
    const int path_cap = c->path_cap;
    c->timing_pending = true;   // event times are read only when asked for (cprrtc_last_timing)
    const QueryOut* out = c->h_out.host<QueryOut>();
    const float* hp = c->h_paths.host<float>();
    const int* hs = c->h_src.host<int>();
    c->last_query_ms = 0.0;
    c->last_kernel_total_ms = 0.0;
    for (int i = 0; i < B; i++) {
        cprrtc_result& r = results[i];
        c->last_query_ms = std::max(c->last_query_ms, out[i].device_ms);
        c->last_kernel_total_ms = std::max(c->last_kernel_total_ms, out[i].total_ms);
        r.setup_code = out[i].setup_code;
        r.status = r.setup_code ? -1 : out[i].status;
        r.path_len = r.status == 0 ? out[i].path_len : 0;
        r.nodes_start = out[i].n_nodes[0];
        r.nodes_goal = out[i].n_nodes[1];
        r.device_ms = out[i].device_ms;
        for (int k = 0; k < CPRRTC_ST_COUNT; k++) r.stats[k] = out[i].stats[k];
        if (paths && r.path_len > 0) {
            const float* src = hp + (size_t)i * path_cap * n;
            double* dst = paths + (size_t)i * path_cap * n;
            for (int k = 0; k < r.path_len * n; k++) dst[k] = src[k];
        }
        if (sources && r.path_len > 1)
            for (int k = 0; k < r.path_len - 1; k++) sources[(size_t)i * path_cap + k] = hs[(size_t)i * path_cap + k];
    }
    return 0;
}

// Batches without waiting: cprrtc_plan_submit launches the per-call sequence
// and returns; cprrtc_plan_wait collects it with the paths packed back to back
// (one pass over the mapped result block, no per-query path_capacity stride).
// A context holds one batch in flight; alternating contexts on one device
// overlap a batch's tail (its slowest queries) with the next batch's start.
int cprrtc_plan_submit(void* p, const cprrtc_params* prm, int B, const double* starts, const double* goals,
                       const int64_t* seeds) {
    Ctx* c = C(p);
    if (!c || !prm || B < 1 || !starts || !goals) return fail(CPRRTC_EARG, "bad argument");
    if (c->inflight) return fail(CPRRTC_EARG, "the context already has a batch in flight");
    if (int rc = check_params(prm)) return rc;
    if (int rc = plan_launch(c, prm, B, starts, goals, seeds, nullptr)) return rc;
    c->inflight = B;
    return 0;
}

int cprrtc_plan_wait(void* p, int B, cprrtc_result* results, int64_t* offsets, double* paths, int32_t* sources,
                     int64_t flat_capacity) {
    Ctx* c = C(p);
    if (!c || B < 1 || !results || !offsets || (flat_capacity > 0 && (!paths || !sources)))
        return fail(CPRRTC_EARG, "bad argument");
    if (c->inflight != B) return fail(CPRRTC_EARG, "no batch of that size in flight on this context");
    c->inflight = 0;
    if (int rc = plan_collect(c, B, results, nullptr, nullptr)) return rc;
    const int n = c->n, path_cap = c->path_cap;
    const float* hp = c->h_paths.host<float>();
    const int* hs = c->h_src.host<int>();
    int64_t off = 0;
    for (int i = 0; i < B; i++) {
        offsets[i] = off;
        off += results[i].path_len;
    }
    offsets[B] = off;
    if (off > flat_capacity) return fail(CPRRTC_ELIMIT, "flat path buffer too small");
    for (int i = 0; i < B; i++) {
        const int L = results[i].path_len;
        if (L <= 0) continue;
        const float* src = hp + (size_t)i * path_cap * n;
        double* dst = paths + (size_t)offsets[i] * n;
        for (int k = 0; k < L * n; k++) dst[k] = src[k];
        const int* ss = hs + (size_t)i * path_cap;
        int32_t* sd = sources + offsets[i];   // L - 1 edge sources, one slot of slack per query
        for (int k = 0; k < L - 1; k++) sd[k] = ss[k];
    }
    return 0;
}

int cprrtc_plan_flat(void* p, const cprrtc_params* prm, int B, const double* starts, const double* goals,
                     const int64_t* seeds, cprrtc_result* results, int64_t* offsets, double* paths,
                     int32_t* sources, int64_t flat_capacity) {
    if (!results || !offsets || (flat_capacity > 0 && (!paths || !sources))) return fail(CPRRTC_EARG, "bad argument");
    if (int rc = cprrtc_plan_submit(p, prm, B, starts, goals, seeds)) return rc;
    return cprrtc_plan_wait(p, B, results, offsets, paths, sources, flat_capacity);
}

int cprrtc_elapsed_ms(void* from, void* to, double* ms) {
    Ctx* a = C(from);
    Ctx* b = C(to);
    if (!a || !b || !ms || a->device != b->device) return fail(CPRRTC_EARG, "bad argument");
    if (a->plan_lean || b->plan_lean)
        return fail(CPRRTC_EARG, "a single-query plan launch records no events (cprrtc_last_timing has its times)");
    float t = 0.f;
    if (int rc = set_device(b)) return rc;
    cudaEventSynchronize(b->ev[3]);
    cudaError_t e = cudaEventElapsedTime(&t, a->ev[0], b->ev[3]);
    if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("cudaEventElapsedTime: ") + cudaGetErrorString(e));
    *ms = t;
    return 0;
}

int cprrtc_plan(void* p, const cprrtc_params* prm, int B, const double* starts, const double* goals,
                const int64_t* seeds, cprrtc_result* results, double* paths, int32_t* sources) {
    Ctx* c = C(p);
    if (!c || !prm || B < 1 || !starts || !goals || !results) return fail(CPRRTC_EARG, "bad argument");
    if (int rc = check_params(prm)) return rc;
    using clk = std::chrono::steady_clock;
    const auto t0 = g_hp_on ? clk::now() : clk::time_point();
    if (int rc = plan_launch(c, prm, B, starts, goals, seeds, nullptr)) return rc;
    if (!g_hp_on) {
        const int rc = plan_collect(c, B, results, paths, sources);
        if (!rc) exact_roots(c, B, starts, goals, results, paths);
        return rc;
    }
    const auto t1 = clk::now();
    if (int rc = wait_results(c, B)) return rc;
    const auto t2 = clk::now();
    const int rc = plan_collect(c, B, results, paths, sources);
    if (!rc) exact_roots(c, B, starts, goals, results, paths);
    const auto t3 = clk::now();
    auto us = [](clk::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
    g_hprof.v[0].push_back(us(t1 - t0) - g_hp_launch_us);
    g_hprof.v[1].push_back(g_hp_launch_us);
    g_hprof.v[2].push_back(us(t2 - t1));
    g_hprof.v[3].push_back(us(t3 - t2));
    return rc;
}

int cprrtc_plan_multi(void* const* ctxs, int n_ctx, const cprrtc_params* prm, int B, const double* starts,
                      const double* goals, const int64_t* seeds, cprrtc_result* results, double* paths,
                      int32_t* sources) {
    if (!ctxs || n_ctx < 1 || !prm || B < 1 || !starts || !goals || !results)
        return fail(CPRRTC_EARG, "bad argument");
    if (int rc = check_params(prm)) return rc;
    std::vector<Ctx*> cs(n_ctx);
    for (int k = 0; k < n_ctx; k++) {
        cs[k] = C(ctxs[k]);
        if (!cs[k]) return fail(CPRRTC_EARG, "NULL context");
        for (int j = 0; j < k; j++)
            if (cs[j] == cs[k]) return fail(CPRRTC_EARG, "a context can appear only once");
        if (cs[k]->n != cs[0]->n) return fail(CPRRTC_EARG, "contexts must share the robot");
    }
    const int n = cs[0]->n;
    const int pc = prm->path_capacity > 0 ? prm->path_capacity : 1024;
    // contiguous shards, launched on every device before any is awaited
    std::vector<int> lo(n_ctx + 1);
    for (int k = 0; k <= n_ctx; k++) lo[k] = (int)((long long)B * k / n_ctx);
    int rc = 0;
    int launched = 0;
    for (int k = 0; k < n_ctx && !rc; k++) {
        const int b = lo[k + 1] - lo[k];
        if (b == 0) continue;
        rc = plan_launch(cs[k], prm, b, starts + (size_t)lo[k] * n, goals + (size_t)lo[k] * n,
                         seeds ? seeds + lo[k] : nullptr, nullptr);
        launched = k + 1;
    }
    for (int k = 0; k < launched; k++) {   // always drain what was launched
        const int b = lo[k + 1] - lo[k];
        if (b == 0) continue;
        int rk = plan_collect(cs[k], b, results + lo[k], paths ? paths + (size_t)lo[k] * pc * n : nullptr,
                              sources ? sources + (size_t)lo[k] * pc : nullptr);
        if (!rc) rc = rk;
    }
    return rc;
}

int cprrtc_plan_race(void* const* ctxs, int n_ctx, const cprrtc_params* prm, const double* start,
                     const double* goal, const int64_t* seeds, cprrtc_result* results, double* paths,
                     int32_t* sources, int32_t* winner) {
    if (!ctxs || n_ctx < 1 || n_ctx > CPRRTC_MAX_RACE || !prm || !start || !goal || !seeds || !results || !winner)
        return fail(CPRRTC_EARG, "bad argument");
    if (int rc = check_params(prm)) return rc;
    std::vector<Ctx*> cs(n_ctx);
    for (int k = 0; k < n_ctx; k++) {
        cs[k] = C(ctxs[k]);
        if (!cs[k]) return fail(CPRRTC_EARG, "NULL context");
        for (int j = 0; j < k; j++)
            if (cs[j] == cs[k]) return fail(CPRRTC_EARG, "a context can race only once");
    }
    // peer access between every pair of distinct devices (NVLink / NVSwitch)
    bool peers = true;
    for (int a = 0; a < n_ctx && peers; a++)
        for (int b = 0; b < n_ctx; b++) {
            const int da = cs[a]->device, db = cs[b]->device;
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) { peers = false; break; }
            CUDA_TRY(cudaSetDevice(da));
            cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(CPRRTC_ECUDA, std::string("peer access: ") + cudaGetErrorString(e));
            cudaGetLastError();
        }
    RaceLink link{};
    link.n = n_ctx;
    // every racer's previous work (its last call's reset kernel included) is
    // drained and every flag word cleared before the first racer launches, so
    // no clear can land after a fast racer's win store
    for (int k = 0; k < n_ctx; k++) {
        if (int rc = set_device(cs[k])) return rc;
        CUDA_TRY(cudaStreamSynchronize(cs[k]->stream));
        if (cs[k]->stream2) CUDA_TRY(cudaStreamSynchronize(cs[k]->stream2));
    }
    if (peers) {
        for (int k = 0; k < n_ctx; k++) {
            if (int rc = set_device(cs[k])) return rc;
            if (int rc = cs[k]->race_flag.ensure(4)) return rc;
            CUDA_TRY(cudaMemset(cs[k]->race_flag.p, 0, 4));
            link.peers[k] = cs[k]->race_flag.as<int>();
        }
        for (int k = 0; k < n_ctx; k++) {
            if (int rc = set_device(cs[k])) return rc;
            CUDA_TRY(cudaDeviceSynchronize());
        }
    } else {
        // one mapped, portable host word owned by racer 0's context (per call
        // state: concurrent races use distinct contexts, hence distinct words)
        if (!cs[0]->race_host) {
            void* h = nullptr;
            if (int rc = set_device(cs[0])) return rc;
            cudaError_t e = cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable);
            if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
            cs[0]->race_host = static_cast<int*>(h);   // UVA: the same address on every device
        }
        *(volatile int*)cs[0]->race_host = 0;
        link.n = 1;
        link.peers[0] = cs[0]->race_host;
    }
    int rc = 0;
    for (int k = 0; k < n_ctx && !rc; k++) {
        link.own = peers ? link.peers[k] : link.peers[0];
        rc = plan_launch(cs[k], prm, 1, start, goal, seeds + k, &link);
    }
    const int pc = prm->path_capacity > 0 ? prm->path_capacity : 1024;
    const int n = cs[0]->n;
    for (int k = 0; k < n_ctx; k++) {   // always drain every launched racer
        int rk = plan_collect(cs[k], 1, results + k, paths ? paths + (size_t)k * pc * n : nullptr,
                              sources ? sources + (size_t)k * pc : nullptr);
        if (!rc) rc = rk;
    }
    if (rc) return rc;
    // winner: the solved racer with the shortest device time
    *winner = -1;
    for (int k = 0; k < n_ctx; k++)
        if (results[k].status == 0 && (*winner < 0 || results[k].device_ms < results[*winner].device_ms))
            *winner = k;
    return 0;
}

int cprrtc_step(void* p, const cprrtc_params* prm, int op, int N, const double* nodes, const int32_t* parents,
                const double* q, int32_t* result, double* new_nodes, int32_t* new_parents, int max_new,
                uint64_t* stats) {
    Ctx* c = C(p);
    if (!c || !prm || (op != 0 && op != 1) || N < 1 || !nodes || !parents || !q || !result || max_new < 0 ||
        (max_new && (!new_nodes || !new_parents)))
        return fail(CPRRTC_EARG, "bad argument");
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = cur_module(c, prm->width, 0, &m)) return rc;
    const int n = c->n;
    int cap = (int)(((long long)N + prm->max_connect_segments + 2 + 127) / 128 * 128);
    if (c->nq_alloc >= 1 && c->cap_alloc >= cap) cap = c->cap_alloc;   // reuse the planner buffers
    const int path_cap = c->path_cap > 0 ? c->path_cap : 1024;
    if (int rc = ensure_plan_buffers(c, c->nq_alloc > 1 ? c->nq_alloc : 1, cap, path_cap)) return rc;
    // tree 0 of query 0 <- the caller's tree (NaN beyond N), its parents, its count
    std::vector<float> soa((size_t)n * cap, NAN);
    for (int i = 0; i < N; i++)
        for (int k = 0; k < n; k++) soa[(size_t)k * cap + i] = (float)nodes[(size_t)i * n + k];
    CUDA_TRY(cudaMemcpyAsync(c->trees.p, soa.data(), soa.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->parents.p, parents, (size_t)N * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->parents.as<int>() + N, 0xff, (size_t)(cap - N) * 4, c->stream));   // -1: unpublished
    QueryState Q;
    CUDA_TRY(cudaMemcpyAsync(&Q, c->qs.p, sizeof Q, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    Q.count[0] = N;
    Q.hwm[0] = cap;          // the next plan() refills the whole tree with NaN
    Q.solved = Q.stop = Q.timed_out = Q.overflow = Q.exhausted = 0;
    Q.setup_code = 0;
    CUDA_TRY(cudaMemcpyAsync(c->qs.p, &Q, sizeof Q, cudaMemcpyHostToDevice, c->stream));
    const double tau = prm->tau_task > 0 ? prm->tau_task : c->tau_task;
    PlanArgs A = make_plan_args(c, prm, 1, cap, tau);
    A.budget_ns = 0;
    std::vector<float> qf(n);
    for (int k = 0; k < n; k++) qf[k] = (float)q[k];
    int rc = upload(c, c->scratch[0], qf.data(), (size_t)n);
    rc = rc ? rc : c->scratch[1].ensure(64);
    rc = rc ? rc : c->scratch[2].ensure(8 * CPRRTC_ST_COUNT);
    if (rc) return rc;
    if (int rc2 = upload_conf(c, m)) return rc2;
    int zero = 0;
    const float* dq = c->scratch[0].as<float>();
    int* dout = c->scratch[1].as<int>();
    unsigned long long* dst = c->scratch[2].as<unsigned long long>();
    void* args[] = {&A, &op, &zero, &dq, &dout, &dst};
    if (int rc2 = launch(c, m, "cp_step_kernel", 1, 1, 32, scene_smem(c, A.scene_g.cull) + m->ws_bytes, args)) return rc2;
    int out[3];
    unsigned long long st[CPRRTC_ST_COUNT];
    download(c, out, c->scratch[1], 3);
    download(c, st, c->scratch[2], CPRRTC_ST_COUNT);
    if (int rc3 = sync(c)) return rc3;
    result[0] = out[0];
    result[1] = out[1];
    result[2] = out[2];
    if (stats)
        for (int i = 0; i < CPRRTC_ST_COUNT; i++) stats[i] = st[i];
    const int added = out[2] - N;
    if (added > max_new) return fail(CPRRTC_ELIMIT, "max_new too small for the appended nodes");
    if (added > 0) {
        std::vector<float> row((size_t)added);
        for (int k = 0; k < n; k++) {
            CUDA_TRY(cudaMemcpy(row.data(), c->trees.as<float>() + (size_t)k * cap + N, (size_t)added * 4,
                                cudaMemcpyDeviceToHost));
            for (int i = 0; i < added; i++) new_nodes[(size_t)i * n + k] = row[i];
        }
        CUDA_TRY(cudaMemcpy(new_parents, c->parents.as<int>() + N, (size_t)added * 4, cudaMemcpyDeviceToHost));
    }
    return 0;
}

int cprrtc_derive_edges(void* p, const cprrtc_params* prm, int n_nodes, const double* nodes, const int32_t* sources,
                        double* dense, int32_t* ok) {
    Ctx* c = C(p);
    if (!c || !prm || n_nodes < 1 || !nodes || (n_nodes > 1 && (!sources || !dense || !ok)))
        return fail(CPRRTC_EARG, "bad argument");
    const int E = n_nodes - 1;
    if (E == 0) return 0;
    if (int rc = set_device(c)) return rc;
    Module* m;
    if (int rc = cur_module(c, prm->width, 0, &m)) return rc;
    const int n = c->n, W = prm->width;
    std::vector<float> nf((size_t)n_nodes * n);
    for (size_t i = 0; i < nf.size(); i++) nf[i] = (float)nodes[i];
    double tau = prm->tau_task > 0 ? prm->tau_task : c->tau_task;
    PlanArgs A = make_plan_args(c, prm, 0, 0, tau);
    int rc = upload(c, c->dense_nodes, nf.data(), nf.size());
    rc = rc ? rc : upload(c, c->scratch[9], sources, (size_t)E);
    rc = rc ? rc : c->dense_buf.ensure((size_t)E * W * n * 4);
    rc = rc ? rc : c->dense_ok.ensure((size_t)E * 4 + 16);
    if (rc) return rc;
    const float* dn = c->dense_nodes.as<float>();
    const int* ds = c->scratch[9].as<int>();
    float* dd = c->dense_buf.as<float>();
    int* dok = c->dense_ok.as<int>();
    void* args[] = {(void*)&E, &A, &dn, &ds, &dd, &dok};
    const int tpc = kThreads / m->G;
    if (int rc2 = upload_conf(c, m)) return rc2;
    if (int rc2 = launch(c, m, "cp_dense_kernel", (E + tpc - 1) / tpc, 1, kThreads, team_smem(c, m, true), args))
        return rc2;
    std::vector<float> tmp((size_t)E * W * n);
    download(c, tmp.data(), c->dense_buf, tmp.size());
    download(c, ok, c->dense_ok, (size_t)E);
    if (int rc3 = sync(c)) return rc3;
    for (size_t i = 0; i < tmp.size(); i++) dense[i] = tmp[i];
    return 0;
}

int cprrtc_clearance(int device, int B, int kind, const double* a, const double* b, double* out) {
    if (B < 0 || (B && (!a || !b || !out)) || (kind != 0 && kind != 1)) return fail(CPRRTC_EARG, "bad argument");
    if (B == 0) return 0;
    CUDA_TRY(cudaSetDevice(device));
    double *da, *db, *dout;
    const size_t bw = kind == 0 ? 6 : 4;
    CUDA_TRY(cudaMalloc(&da, (size_t)B * 4 * 8));
    CUDA_TRY(cudaMalloc(&db, (size_t)B * bw * 8));
    CUDA_TRY(cudaMalloc(&dout, (size_t)B * 8));
    cudaMemcpy(da, a, (size_t)B * 4 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b, (size_t)B * bw * 8, cudaMemcpyHostToDevice);
    cudaError_t e = cprrtc::launch_clearance(B, kind, da, db, dout, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, (size_t)B * 8, cudaMemcpyDeviceToHost);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dout);
    if (e != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("clearance: ") + cudaGetErrorString(e));
    return 0;
}

int cprrtc_damped_step(int device, int B, int m, int n, const double* J, const double* e, double lam, double* step,
                       int32_t* ok) {
    if (B < 0 || m < 1 || m > 5 || n < 1 || n > 32 || (B && (!J || !e || !step || !ok)))
        return fail(CPRRTC_EARG, "bad argument (1 <= m <= 5, 1 <= n <= 32)");
    if (B == 0) return 0;
    CUDA_TRY(cudaSetDevice(device));
    double *dJ, *de, *ds;
    int32_t* dok;
    CUDA_TRY(cudaMalloc(&dJ, (size_t)B * m * n * 8));
    CUDA_TRY(cudaMalloc(&de, (size_t)B * m * 8));
    CUDA_TRY(cudaMalloc(&ds, (size_t)B * n * 8));
    CUDA_TRY(cudaMalloc(&dok, (size_t)B * 4));
    cudaMemcpy(dJ, J, (size_t)B * m * n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(de, e, (size_t)B * m * 8, cudaMemcpyHostToDevice);
    cudaError_t err = cprrtc::launch_damped_step(B, m, n, dJ, de, lam, ds, dok, 0);
    if (err == cudaSuccess) err = cudaMemcpy(step, ds, (size_t)B * n * 8, cudaMemcpyDeviceToHost);
    if (err == cudaSuccess) err = cudaMemcpy(ok, dok, (size_t)B * 4, cudaMemcpyDeviceToHost);
    cudaFree(dJ);
    cudaFree(de);
    cudaFree(ds);
    cudaFree(dok);
    if (err != cudaSuccess) return fail(CPRRTC_ECUDA, std::string("damped_step: ") + cudaGetErrorString(err));
    return 0;
}

}  // extern "C"
