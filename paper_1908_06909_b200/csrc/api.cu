// api.cu -- the C ABI of libtetproj (include/tetproj.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace tetproj;

struct tet_mesh {
    int device = 0;
    // walk shape hint: the last call with statistics saw > 5 % exact
    // fallbacks per crossing (kernels.cu TraceShape<., true>)
    std::atomic<int> exact_heavy{0};
    uint32_t flags = 0;
    HostMesh host;      // keeps grid parameters (arrays freed after upload)
    DevMesh dev;
    void* d_rec = nullptr;
    void* d_tag16 = nullptr;
    void* d_tnode = nullptr;
    void* d_vtx = nullptr;
    void* d_hull = nullptr;
    void* d_perm = nullptr;
    void* d_bvh_nodes = nullptr;
    void* d_bvh_faces = nullptr;
    void* d_rtree = nullptr;
    // private stream-ordered pool for per-call scratch: freed scratch stays
    // cached across this mesh's calls (no re-allocation inside timed calls)
    // and is returned to the device at tet_mesh_destroy; the device's default
    // pool -- shared with the rest of the process -- is never touched
    cudaMemPool_t pool = nullptr;
    int64_t bytes = 0;
    int64_t tag16_bytes = 0, rtree_nodes = 0, bvh_nodes = 0;
    // kernel timing (tet_set_kernel_timing)
    struct TimerRec { int kind; cudaEvent_t a, b; };
    std::mutex tmu;
    bool timing = false;
    std::vector<TimerRec> pending;
    std::vector<cudaEvent_t> spare;
    double ms[TET_K_COUNT] = {0, 0, 0, 0};
    int64_t launches[TET_K_COUNT] = {0, 0, 0, 0};
    // side streams of the calls (second walk stream, host-copy stream),
    // created once and reused: a cudaStreamCreate inside a timed call could
    // stall the host while the GPU idles (seen as a ~4-ms gap in a first call)
    std::mutex smu;
    std::vector<cudaStream_t> streams;
    cudaError_t take_stream(cudaStream_t& out) {
        {
            std::lock_guard<std::mutex> g(smu);
            if (!streams.empty()) {
                out = streams.back();
                streams.pop_back();
                return cudaSuccess;
            }
        }
        return cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking);
    }
    void give_stream(cudaStream_t st) {   // pending work on it is fine: later use is ordered after
        std::lock_guard<std::mutex> g(smu);
        streams.push_back(st);
    }
};

// A scan bound to a mesh (tet_plan_create): the snapped geometry tables and
// the entry map of every ray, computed once and shared by the plan's calls.
struct tet_plan {
    tet_mesh* m = nullptr;
    tet_geometry g{};
    std::vector<double> vecs;
    tet_options opt{};
    bool has_opt = false;
    std::vector<tetproj::AngleGeom> ang;
    std::vector<tetproj::AngleAux> aux;
    tetproj::AngleGeom* d_ang = nullptr;
    tetproj::AngleAux* d_aux = nullptr;
    int* d_entry = nullptr;                    // [n_angles][n_v][n_u], -1 = miss
    unsigned long long* d_stats = nullptr;     // the entry finder's counters
};

namespace {

thread_local std::string g_err;

tet_status fail(tet_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

tet_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? TET_E_NOMEM : TET_E_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(call)                                             \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
    } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Is `p` device memory of `dev`?  (host pinned / pageable -> false)
bool is_device_ptr(const void* p, int dev, bool& wrong_device) {
    wrong_device = false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
        if (at.type == cudaMemoryTypeDevice && at.device != dev) wrong_device = true;
        return true;
    }
    return false;
}

// Scratch allocated stream-ordered from the mesh's private pool.
struct Scratch {
    cudaStream_t s;
    cudaMemPool_t pool;
    std::vector<void*> ptrs;
    Scratch(cudaStream_t st, cudaMemPool_t p) : s(st), pool(p) {}
    cudaError_t alloc(void** p, size_t n) {
        cudaError_t e = cudaMallocFromPoolAsync(p, n ? n : 16, pool, s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
};

cudaError_t make_pool(int dev, cudaMemPool_t* pool) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaError_t e = cudaMemPoolCreate(pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;   // keep this mesh's freed scratch until destroy
    return cudaMemPoolSetAttribute(*pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// Entry: only the entry finder, into a plan's entry map (tet_plan_create)
enum class Op { Forward, Backward, BackwardF64, Entry };

cudaEvent_t take_event(tet_mesh* m) {
    cudaEvent_t e = nullptr;
    if (!m->spare.empty()) {
        e = m->spare.back();
        m->spare.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}

// Records CUDA events around one kernel launch when timing is enabled.
struct KernelTimer {
    tet_mesh* m;
    int kind;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    KernelTimer(tet_mesh* mm, int k, cudaStream_t st) : m(mm), kind(k), s(st) {
        if (!m->timing) return;
        std::lock_guard<std::mutex> g(m->tmu);
        a = take_event(m);
        cudaEventRecord(a, s);
    }
    ~KernelTimer() {
        if (!a) return;
        std::lock_guard<std::mutex> g(m->tmu);
        cudaEvent_t b = take_event(m);
        cudaEventRecord(b, s);
        m->pending.push_back({kind, a, b});
    }
};

// Second walk stream of one call: consecutive angle chunks alternate between
// the caller's stream and this one (with their own entry buffers), so chunk
// k+1's entry finder and the head of its walk overlap the tail of chunk k's
// walk -- a serialised chunk boundary cost ~0.2 ms (c3, profiles/README.md).
struct AuxStream {
    tet_mesh* m;
    cudaStream_t main, s = nullptr;
    cudaError_t err = cudaSuccess;
    static cudaError_t wait(cudaStream_t waiter, cudaStream_t on) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r != cudaSuccess) return r;
        r = cudaEventRecord(e, on);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(waiter, e, 0);
        cudaEventDestroy(e);   // released once the recorded work completes
        return r;
    }
    // `on`: everything queued on the caller's stream so far is visible to it
    AuxStream(tet_mesh* mesh, cudaStream_t st, bool on) : m(mesh), main(st) {
        if (!on) return;
        err = m->take_stream(s);
        if (err != cudaSuccess) {
            s = nullptr;
            return;
        }
        err = wait(s, main);
    }
    cudaStream_t get(size_t k) const { return (s && (k & 1)) ? s : main; }
    cudaError_t join() const { return s ? wait(main, s) : cudaSuccess; }
    ~AuxStream() {   // the caller's stream (and the scratch frees on it) waits for it
        if (!s) return;
        wait(main, s);
        m->give_stream(s);
    }
};

// Side stream for the pipelined host copies of one call, with its events.
struct CopyStream {
    tet_mesh* m;
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaError_t err = cudaSuccess;
    CopyStream(tet_mesh* mesh, bool on) : m(mesh) {
        if (!on) return;
        err = m->take_stream(s);
        if (err != cudaSuccess) s = nullptr;
    }
    cudaError_t event(cudaEvent_t& e) {
        cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r == cudaSuccess) ev.push_back(e);
        return r;
    }
    // copy stream waits for everything queued on `on` so far
    cudaError_t after(cudaStream_t on) {
        cudaEvent_t e;
        cudaError_t r = event(e);
        if (r == cudaSuccess) r = cudaEventRecord(e, on);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(s, e, 0);
        ev.pop_back();          // only the mark() events are indexed by chunk
        cudaEventDestroy(e);    // released once the recorded work completes
        return r;
    }
    // event after the last queued copy (ev[k] for the k-th mark)
    cudaError_t mark() {
        cudaEvent_t e;
        cudaError_t r = event(e);
        return r == cudaSuccess ? cudaEventRecord(e, s) : r;
    }
    // `on` waits for every copy queued so far
    cudaError_t join(cudaStream_t on) {
        cudaEvent_t e;
        cudaError_t r = event(e);
        if (r == cudaSuccess) r = cudaEventRecord(e, s);
        return r == cudaSuccess ? cudaStreamWaitEvent(on, e, 0) : r;
    }
    ~CopyStream() {   // before the scratch it reads is released (also on error paths)
        if (s) cudaStreamSynchronize(s);
        for (auto e : ev) cudaEventDestroy(e);
        if (s) m->give_stream(s);
    }
};

// Shared driver: geometry prep, chunking over angles, entry finder, walker.
// With a plan, the geometry tables and the entry map are the plan's (op
// Entry computes that map; the other ops skip the entry finder).
tet_status run(tet_mesh_t m, const tet_geometry* g, const float* in, void* out, int accumulate,
               Op op, void* stream, tet_stats* st, const tet_options* opt = nullptr,
               tet_plan* plan = nullptr) {
    if (!m) return fail(TET_E_ARG, "null mesh");
    const bool entry_only = op == Op::Entry;
    const bool use_plan = plan && !entry_only;
    const int mode = opt ? opt->traversal : TET_TRAVERSE_EXACT;
    const int entry_mode = opt ? opt->entry : TET_ENTRY_RASTER;
    if (entry_mode != TET_ENTRY_RASTER && entry_mode != TET_ENTRY_BVH &&
        entry_mode != TET_ENTRY_RTREE)
        return fail(TET_E_ARG, "unknown entry finder");
    if (mode < TET_TRAVERSE_EXACT || mode > TET_TRAVERSE_MT_F32)
        return fail(TET_E_ARG, "unknown traversal mode");
    MtOptions mto;
    if (opt && mode != TET_TRAVERSE_EXACT) {
        if (!(opt->eps0 > 0) || !(opt->eps_growth > 1) || opt->max_escalations < 0)
            return fail(TET_E_ARG, "bad MT options (eps0 > 0, eps_growth > 1, max_escalations >= 0)");
        mto.eps0 = opt->eps0;
        mto.eps_growth = opt->eps_growth;
        mto.max_escalations = opt->max_escalations;
    }
    if (!g || (!entry_only && (!in || !out))) return fail(TET_E_ARG, "null argument");
    if (entry_only && !plan) return fail(TET_E_ARG, "entry map without a plan");
    std::vector<AngleGeom> ang_own;
    std::vector<AngleAux> aux_own;
    if (!plan) {
        std::string err;
        tet_status rs = prepare_geometry(m->host, g, ang_own, aux_own, err);
        if (rs != TET_OK) return fail(rs, err);
    }
    const std::vector<AngleGeom>& ang = plan ? plan->ang : ang_own;
    const std::vector<AngleAux>& aux = plan ? plan->aux : aux_own;
    DeviceGuard guard(m->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nrays = (int64_t)g->n_angles * g->n_v * g->n_u;
    const int64_t nt = m->dev.nt;
    bool wd_in = false, wd_out = false;
    const bool dev_in = entry_only || is_device_ptr(in, m->device, wd_in);
    const bool dev_out = entry_only || is_device_ptr(out, m->device, wd_out);
    if (wd_in || wd_out) return fail(TET_E_ARG, "device pointer on another device than the mesh");
    if (op == Op::BackwardF64 && !dev_out) return fail(TET_E_ARG, "tet_backproject_f64 needs a device accumulator");
    const size_t in_bytes = (op == Op::Forward ? nt : nrays) * sizeof(float);
    const size_t out_elems = (op == Op::Forward ? nrays : nt);
    const bool strict = (m->flags & TET_F_STRICT) != 0;
    const bool need_stats = !entry_only && (st || strict);
    unsigned long long hs[ST_COUNT] = {0};
    {
        Scratch sc(s, m->pool);  // released (stream-ordered) at the end of this scope
        // --- stage host inputs / outputs through device memory.  The
        // per-ray host arrays (y of a backprojection, proj of a projection)
        // move chunk by chunk on a copy stream, overlapped with the tracing
        // of the neighbouring chunks; the per-tet ones (mu, x) are small.
        const bool pipe_in = !dev_in && op != Op::Forward;
        const bool pipe_out = !dev_out && op == Op::Forward;
        CopyStream cs(m, pipe_in || pipe_out);
        if (cs.err != cudaSuccess) return cuda_fail(cs.err, "copy stream");
        const float* d_in = in;
        if (!dev_in) {
            void* p;
            CU(sc.alloc(&p, in_bytes));
            if (!pipe_in) CU(cudaMemcpyAsync(p, in, in_bytes, cudaMemcpyHostToDevice, s));
            d_in = (const float*)p;
        }
        void* d_out = out;
        if (!dev_out) {
            CU(sc.alloc(&d_out, out_elems * sizeof(float)));
            if (op == Op::Backward && accumulate)
                CU(cudaMemcpyAsync(d_out, out, out_elems * sizeof(float), cudaMemcpyHostToDevice, s));
        }
        // --- geometry tables (a plan's are on the device already)
        AngleGeom* d_ang;
        AngleAux* d_aux;
        unsigned long long* d_stats;
        if (plan) {
            d_ang = plan->d_ang;
            d_aux = plan->d_aux;
        } else {
            CU(sc.alloc((void**)&d_ang, sizeof(AngleGeom) * ang.size()));
            CU(sc.alloc((void**)&d_aux, sizeof(AngleAux) * aux.size()));
            CU(cudaMemcpyAsync(d_ang, ang.data(), sizeof(AngleGeom) * ang.size(), cudaMemcpyHostToDevice, s));
            CU(cudaMemcpyAsync(d_aux, aux.data(), sizeof(AngleAux) * aux.size(), cudaMemcpyHostToDevice, s));
        }
        if (entry_only) {
            d_stats = plan->d_stats;
            CU(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * ST_COUNT, s));
        } else {
            CU(sc.alloc((void**)&d_stats, sizeof(unsigned long long) * ST_COUNT));
            if (use_plan)   // the counters start from the entry finder's (conflicts, exact)
                CU(cudaMemcpyAsync(d_stats, plan->d_stats, sizeof(unsigned long long) * ST_COUNT,
                                   cudaMemcpyDeviceToDevice, s));
            else
                CU(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * ST_COUNT, s));
        }
        // --- per-op buffers
        float* mu_int = nullptr;
        double* acc = nullptr;
        if (entry_only) {
        } else if (op == Op::Forward) {
            CU(sc.alloc((void**)&mu_int, nt * sizeof(float)));
            KernelTimer kt(m, TET_K_PERMUTE, s);
            CU(launch_gather_mu(m->dev, d_in, mu_int, s));
        } else {
            CU(sc.alloc((void**)&acc, nt * sizeof(double)));
            CU(cudaMemsetAsync(acc, 0, nt * sizeof(double), s));
        }
        // --- angle chunks bound the entry-map scratch (<= 2^26 rays per chunk).
        // With host copies pipelined, the first chunk's copy-in and the last
        // chunk's copy-out are exposed while every chunk costs a fixed
        // overhead: about an eighth of the call's rays per chunk, within
        // [2^21, 2^25] (c3, 94 M rays: 1.568e11 at 2^23, 1.573e11 at 2^24,
        // 1.527e11 at 2^25; c5, 755 M rays: 1.610e11 at 2^23, 1.638e11 at 2^25;
        // c2, 5.9 M rays: 1.364e11 at 2^22, 1.477e11 at 2^21, 1.493e11 at 2^20;
        // c4a, 4.2 M rays with latency-bound walks: 8.99e9 at 2^22, 9.81e9 at
        // 2^21, 6.95e9 at 2^20 crossings/s end to end; TETPROJ_PIPE_CHUNK_LOG
        // forces a size)
        const int64_t per_angle = (int64_t)g->n_v * g->n_u;
        static const int pipe_log = [] {   // A/B knob for the host-buffer pipeline
            const char* e = getenv("TETPROJ_PIPE_CHUNK_LOG");
            const int v = e ? atoi(e) : 0;
            return v >= 16 && v <= 26 ? v : 0;
        }();
        const int64_t pipe_rays = pipe_log ? (1LL << pipe_log)
                                           : std::max<int64_t>(1LL << 21, std::min<int64_t>(1LL << 25, nrays / 8));
        const int64_t max_chunk_rays = (pipe_in || pipe_out) ? pipe_rays : (1LL << 26);
        // and <= kUniMaxAngles angles (one walker launch per chunk)
        const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(g->n_angles, kUniMaxAngles),
                                                                      max_chunk_rays / per_angle));
        // Chunk schedule (angle counts).  With host buffers the first chunk's
        // copy-in (backprojection) and the last chunk's copy-out (projection)
        // cannot overlap any tracing, so those ends are tapered: c/4, c/4, c/2
        // at the head and c/2, c/4, c/4 at the tail (TETPROJ_PIPE_TAPER=0: all c).
        static const int taper_env = [] {
            const char* e = getenv("TETPROJ_PIPE_TAPER");
            return e ? atoi(e) : 1;
        }();
        std::vector<int> sizes;
        {
            int rem = g->n_angles;
            const bool taper = taper_env && g->n_angles > 2 * chunk;
            std::vector<int> head, tail;
            if (taper && pipe_in) head = {std::max(1, chunk / 4), std::max(1, chunk / 4), std::max(1, chunk / 2)};
            if (taper && pipe_out) tail = {std::max(1, chunk / 2), std::max(1, chunk / 4), std::max(1, chunk / 4)};
            int tail_total = 0;
            for (int t : tail) tail_total += t;
            for (int h : head)
                if (rem > tail_total) { const int t = std::min(h, rem - tail_total); sizes.push_back(t); rem -= t; }
            while (rem > tail_total) { const int t = std::min(chunk, rem - tail_total); sizes.push_back(t); rem -= t; }
            for (int t : tail)
                if (rem > 0) { const int u = std::min(t, rem); sizes.push_back(u); rem -= u; }
        }
        if (pipe_in) {   // all y chunks are queued at once; chunk k's trace waits for its copy
            CU(cs.after(s));
            int a0 = 0;
            for (int na : sizes) {
                const size_t off = (size_t)a0 * per_angle;
                const size_t n = (size_t)na * per_angle;
                CU(cudaMemcpyAsync((float*)d_in + off, (const float*)in + off, n * sizeof(float),
                                   cudaMemcpyHostToDevice, cs.s));
                CU(cs.mark());
                a0 += na;
            }
        }
        size_t chunk_idx = 0;
        const int n_chunks = (int)sizes.size();
        const int nbuf = n_chunks > 1 ? 2 : 1;
        int* entry[2] = {nullptr, nullptr};
        void* entry_scratch[2] = {nullptr, nullptr};
        for (int b = 0; b < nbuf && !use_plan; ++b) {
            if (!entry_only) CU(sc.alloc((void**)&entry[b], sizeof(int) * per_angle * chunk));
            CU(sc.alloc(&entry_scratch[b], entry_scratch_bytes(m->dev, chunk)));
        }
        // chunk k runs on ws.get(k) with entry buffer k % 2 (the chunk k-2
        // that used it before is earlier on the same stream)
        static const int heavy_env = [] {   // TETPROJ_EXACT_HEAVY=0/1 forces the shape
            const char* e = getenv("TETPROJ_EXACT_HEAVY");
            return e ? atoi(e) : -1;
        }();
        const int heavy = heavy_env >= 0 ? (heavy_env != 0) : m->exact_heavy.load();
        AuxStream ws(m, s, n_chunks > 1);
        if (ws.err != cudaSuccess) return cuda_fail(ws.err, "walk stream");
        int a0 = 0;
        for (const int na : sizes) {
            cudaStream_t sk = ws.get(chunk_idx);
            const size_t off = (size_t)a0 * per_angle;
            int* ent = plan ? plan->d_entry + off : entry[chunk_idx % nbuf];
            LaunchChunk c{d_ang + a0, ang.data() + a0, d_aux + a0, g->beam, na, g->n_v, g->n_u};
            c.exact_heavy = heavy;
            if (!use_plan) {
                CU(cudaMemsetAsync(ent, 0xff, sizeof(int) * per_angle * na, sk));
                KernelTimer kt(m, TET_K_ENTRY, sk);
                if (entry_mode == TET_ENTRY_BVH)
                    CU(launch_entry_bvh(m->dev, c, ent, d_stats, sk));
                else if (entry_mode == TET_ENTRY_RTREE)
                    CU(launch_entry_rtree(m->dev, c, ent, d_stats, sk));
                else
                    CU(launch_entry(m->dev, c, ent, entry_scratch[chunk_idx % nbuf], d_stats, sk));
            }
            if (entry_only) {
                ++chunk_idx;
                a0 += na;
                continue;
            }
            const bool fwd = op == Op::Forward;
            if (pipe_in) CU(cudaStreamWaitEvent(sk, cs.ev[chunk_idx], 0));
            ++chunk_idx;
            if (mode != TET_TRAVERSE_EXACT) {
                KernelTimer kt(m, fwd ? TET_K_FORWARD : TET_K_BACKWARD, sk);
                CU(launch_mt(m->dev, c, !fwd, mode == TET_TRAVERSE_MT_F32, mto, ent, mu_int,
                             fwd ? (float*)d_out + off : nullptr, fwd ? nullptr : d_in + off, acc,
                             d_stats, sk));
            } else if (fwd) {
                KernelTimer kt(m, TET_K_FORWARD, sk);
                CU(launch_forward(m->dev, c, ent, mu_int, (float*)d_out + off, d_stats, sk));
            } else {
                KernelTimer kt(m, TET_K_BACKWARD, sk);
                CU(launch_backward(m->dev, c, ent, d_in + off, acc, d_stats, sk));
            }
            if (pipe_out) {   // this chunk's projections go home while the next one traces
                CU(cs.after(sk));
                CU(cudaMemcpyAsync((float*)out + off, (float*)d_out + off,
                                   (size_t)na * per_angle * sizeof(float), cudaMemcpyDeviceToHost,
                                   cs.s));
            }
            a0 += na;
        }
        CU(ws.join());
        if (pipe_out) CU(cs.join(s));
        if (op == Op::Backward) {
            KernelTimer kt(m, TET_K_PERMUTE, s);
            CU(launch_scatter_x(m->dev, acc, (float*)d_out, accumulate, s));
        }
        if (op == Op::BackwardF64) {
            KernelTimer kt(m, TET_K_PERMUTE, s);
            CU(launch_scatter_acc(m->dev, acc, (double*)d_out, s));
        }
        if (!dev_out && !pipe_out)
            CU(cudaMemcpyAsync(out, d_out, out_elems * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (need_stats) CU(cudaMemcpyAsync(hs, d_stats, sizeof hs, cudaMemcpyDeviceToHost, s));
        CU(cudaGetLastError());
    }
    if (need_stats || !dev_out || !dev_in) CU(cudaStreamSynchronize(s));
    if (need_stats && mode == TET_TRAVERSE_EXACT && hs[ST_CROSS] > 0)
        m->exact_heavy.store(hs[ST_EXACT] * 20 > hs[ST_CROSS] ? 1 : 0);
    if (st) {
        std::memset(st, 0, sizeof *st);
        st->rays = (uint64_t)nrays;
        st->rays_hit = hs[ST_HIT];
        st->crossings = hs[ST_CROSS];
        st->lost = hs[ST_LOST];
        st->stuck = hs[ST_STUCK];
        st->exact_fallbacks = hs[ST_EXACT];
        st->entry_conflicts = hs[ST_CONFLICT];
        st->max_crossings_per_ray = (uint32_t)hs[ST_MAXC];
        st->escalations = hs[ST_ESC];
    }
    if (strict && (hs[ST_LOST] || hs[ST_STUCK] || hs[ST_CONFLICT]))
        return fail(TET_E_RAYS, "lost / stuck / conflicting rays (TET_F_STRICT)");
    return TET_OK;
}

}  // namespace

extern "C" {

const char* tet_last_error(void) { return g_err.c_str(); }

tet_status tet_mesh_create(const double* verts, int64_t n_verts, const int32_t* tets,
                           const int32_t* nbrs, int64_t n_tets, const int32_t* bfaces,
                           int64_t n_bfaces, int device, uint32_t flags, tet_mesh_t* out) {
    if (!out) return fail(TET_E_ARG, "null output handle");
    *out = nullptr;
    // host-side validation first: mesh errors are reported as such even on a
    // machine without a usable device
    tet_mesh* m = new tet_mesh();
    std::string err;
    tet_status s = prepare_mesh(verts, n_verts, tets, nbrs, n_tets, bfaces, n_bfaces, flags,
                                m->host, err);
    if (s != TET_OK) {
        delete m;
        return fail(s, err);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        delete m;
        return fail(TET_E_CUDA, "no such CUDA device: " + std::to_string(device));
    }
    m->device = device;
    m->flags = flags;
    DeviceGuard guard(device);
    HostMesh& H = m->host;
    auto up = [&](void** d, const void* h, size_t n) -> cudaError_t {
        cudaError_t e = cudaMalloc(d, n ? n : 16);
        if (e == cudaSuccess && n) e = cudaMemcpy(*d, h, n, cudaMemcpyHostToDevice);
        m->bytes += (int64_t)n;
        return e;
    };
    cudaError_t e = make_pool(device, &m->pool);
    if (e == cudaSuccess) e = up(&m->d_rec, H.rec.data(), H.rec.size() * 4);
    // FT16 walk unless the mesh exceeds its encoding or TETPROJ_WALKER=rec
    // asks for the 32-B-record walk (A/B measurements)
    const char* wk = std::getenv("TETPROJ_WALKER");
    const bool ft16 = H.ft16 && !(wk && std::string(wk) == "rec");
    if (e == cudaSuccess && ft16) e = up(&m->d_tag16, H.tag16.data(), H.tag16.size() * 4);
    m->tag16_bytes = ft16 ? (int64_t)H.tag16.size() * 4 : 0;
    m->rtree_nodes = (int64_t)H.rtree_nodes.size() / 72;
    m->bvh_nodes = (int64_t)H.bvh_nodes.size() / 8;
    if (e == cudaSuccess) e = up(&m->d_tnode, H.tnode.data(), H.tnode.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_vtx, H.vtx.data(), H.vtx.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_hull, H.hull.data(), H.hull.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_perm, H.perm.data(), H.perm.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_bvh_nodes, H.bvh_nodes.data(), H.bvh_nodes.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_bvh_faces, H.bvh_faces.data(), H.bvh_faces.size() * 4);
    if (e == cudaSuccess) e = up(&m->d_rtree, H.rtree_nodes.data(), H.rtree_nodes.size() * 4);
    if (e != cudaSuccess) {
        tet_mesh_destroy(m);
        return cuda_fail(e, "tet_mesh_create upload");
    }
    m->dev.rec = (const int4*)m->d_rec;
    m->dev.tag16 = (const int4*)m->d_tag16;
    m->dev.tnode = (const int4*)m->d_tnode;
    m->dev.vtx = (const int4*)m->d_vtx;
    m->dev.hull = (const int2*)m->d_hull;
    m->dev.perm = (const int*)m->d_perm;
    m->dev.bvh_nodes = (const int4*)m->d_bvh_nodes;
    m->dev.bvh_faces = (const int4*)m->d_bvh_faces;
    m->dev.rtree = (const int*)m->d_rtree;
    m->dev.nv = H.nv;
    m->dev.nt = H.nt;
    m->dev.nb = H.nb;
    m->dev.g = H.g;
    m->dev.rmax = H.rmax;
    for (int i = 0; i < 3; ++i) m->dev.C[i] = H.C[i];
    {   // L2 persistence for the face tags (TETPROJ_L2_PERSIST=1): carve out the
        // device's persisting L2 and size the window to the records
        const char* ev = std::getenv("TETPROJ_L2_PERSIST");
        if (ev && ev[0] == '1') {
            int max_persist = 0, max_window = 0;
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
            cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
            // the walked table: FT16 tags (64 B per tet) or the records (32 B)
            const size_t table_bytes = (size_t)H.nt * (H.ft16 ? 64 : 32);
            if (max_persist > 0 && max_window > 0) {
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
                m->dev.l2_window_bytes = std::min(table_bytes, (size_t)max_window);
                m->dev.l2_hit_ratio = std::min(1.0, (double)max_persist / (double)m->dev.l2_window_bytes);
            }
        }
    }
    // host copies are no longer needed
    std::vector<int32_t>().swap(H.rec);
    std::vector<int32_t>().swap(H.tag16);
    std::vector<int32_t>().swap(H.tnode);
    std::vector<int32_t>().swap(H.vtx);
    std::vector<int32_t>().swap(H.hull);
    std::vector<int32_t>().swap(H.perm);
    std::vector<int32_t>().swap(H.bvh_nodes);
    std::vector<int32_t>().swap(H.bvh_faces);
    std::vector<int32_t>().swap(H.rtree_nodes);
    *out = m;
    return TET_OK;
}

tet_status tet_mesh_destroy(tet_mesh_t m) {
    if (!m) return TET_OK;
    DeviceGuard guard(m->device);
    for (auto& r : m->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : m->spare) cudaEventDestroy(e);
    for (auto st : m->streams) cudaStreamDestroy(st);
    cudaFree(m->d_rec);
    cudaFree(m->d_tag16);
    cudaFree(m->d_tnode);
    cudaFree(m->d_vtx);
    cudaFree(m->d_hull);
    cudaFree(m->d_perm);
    cudaFree(m->d_bvh_nodes);
    cudaFree(m->d_bvh_faces);
    cudaFree(m->d_rtree);
    // returned to the device once the last stream-ordered free has run
    if (m->pool) cudaMemPoolDestroy(m->pool);
    delete m;
    return TET_OK;
}

tet_status tet_project(tet_mesh_t m, const tet_geometry* g, const float* mu, float* proj,
                       void* cuda_stream, tet_stats* st) {
    return run(m, g, mu, proj, 0, Op::Forward, cuda_stream, st);
}

tet_status tet_project_ex(tet_mesh_t m, const tet_geometry* g, const float* mu, float* proj,
                          const tet_options* opt, void* cuda_stream, tet_stats* st) {
    return run(m, g, mu, proj, 0, Op::Forward, cuda_stream, st, opt);
}

tet_status tet_backproject_ex(tet_mesh_t m, const tet_geometry* g, const float* proj, float* x,
                              int accumulate, const tet_options* opt, void* cuda_stream,
                              tet_stats* st) {
    return run(m, g, proj, x, accumulate, Op::Backward, cuda_stream, st, opt);
}

tet_status tet_backproject(tet_mesh_t m, const tet_geometry* g, const float* proj, float* x,
                           int accumulate, void* cuda_stream, tet_stats* st) {
    return run(m, g, proj, x, accumulate, Op::Backward, cuda_stream, st);
}

tet_status tet_backproject_f64(tet_mesh_t m, const tet_geometry* g, const float* proj,
                               double* acc, void* cuda_stream, tet_stats* st) {
    return run(m, g, proj, acc, 1, Op::BackwardF64, cuda_stream, st);
}

tet_status tet_plan_create(tet_mesh_t m, const tet_geometry* g, const tet_options* opt,
                           void* cuda_stream, tet_plan_t* out) {
    if (!out) return fail(TET_E_ARG, "null argument");
    *out = nullptr;
    if (!m || !g || !g->vecs) return fail(TET_E_ARG, "null argument");
    if (opt && opt->entry != TET_ENTRY_RASTER && opt->entry != TET_ENTRY_BVH &&
        opt->entry != TET_ENTRY_RTREE)
        return fail(TET_E_ARG, "unknown entry finder");
    if (opt && (opt->traversal < TET_TRAVERSE_EXACT || opt->traversal > TET_TRAVERSE_MT_F32))
        return fail(TET_E_ARG, "unknown traversal mode");
    tet_plan* p = new tet_plan;
    p->m = m;
    p->g = *g;
    if (g->n_angles > 0) p->vecs.assign(g->vecs, g->vecs + (size_t)g->n_angles * 12);
    p->g.vecs = p->vecs.data();
    if (opt) {
        p->opt = *opt;
        p->has_opt = true;
    }
    std::string err;
    tet_status rs = prepare_geometry(m->host, g, p->ang, p->aux, err);
    if (rs != TET_OK) {
        delete p;
        return fail(rs, err);
    }
    DeviceGuard guard(m->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const size_t nrays = (size_t)g->n_angles * g->n_v * g->n_u;
    auto alloc = [&](void** q, size_t n) { return cudaMallocFromPoolAsync(q, n ? n : 16, m->pool, s); };
    cudaError_t e = alloc((void**)&p->d_ang, sizeof(AngleGeom) * p->ang.size());
    if (e == cudaSuccess) e = alloc((void**)&p->d_aux, sizeof(AngleAux) * p->aux.size());
    if (e == cudaSuccess) e = alloc((void**)&p->d_entry, sizeof(int) * nrays);
    if (e == cudaSuccess) e = alloc((void**)&p->d_stats, sizeof(unsigned long long) * ST_COUNT);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->d_ang, p->ang.data(), sizeof(AngleGeom) * p->ang.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->d_aux, p->aux.data(), sizeof(AngleAux) * p->aux.size(), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
        tet_plan_destroy(p, cuda_stream);
        return cuda_fail(e, "tet_plan_create");
    }
    rs = run(m, &p->g, nullptr, nullptr, 0, Op::Entry, cuda_stream, nullptr,
             p->has_opt ? &p->opt : nullptr, p);
    if (rs != TET_OK) {
        const std::string msg = g_err;
        tet_plan_destroy(p, cuda_stream);
        return fail(rs, msg);
    }
    *out = p;
    return TET_OK;
}

tet_status tet_plan_destroy(tet_plan_t p, void* cuda_stream) {
    if (!p) return TET_OK;
    DeviceGuard guard(p->m->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    for (void* q : {(void*)p->d_ang, (void*)p->d_aux, (void*)p->d_entry, (void*)p->d_stats})
        if (q) cudaFreeAsync(q, s);
    delete p;
    return TET_OK;
}

tet_status tet_plan_project(tet_plan_t p, const float* mu, float* proj, void* cuda_stream,
                            tet_stats* st) {
    if (!p) return fail(TET_E_ARG, "null plan");
    return run(p->m, &p->g, mu, proj, 0, Op::Forward, cuda_stream, st,
               p->has_opt ? &p->opt : nullptr, p);
}

tet_status tet_plan_backproject(tet_plan_t p, const float* proj, float* x, int accumulate,
                                void* cuda_stream, tet_stats* st) {
    if (!p) return fail(TET_E_ARG, "null plan");
    return run(p->m, &p->g, proj, x, accumulate, Op::Backward, cuda_stream, st,
               p->has_opt ? &p->opt : nullptr, p);
}

tet_status tet_plan_backproject_f64(tet_plan_t p, const float* proj, double* acc,
                                    void* cuda_stream, tet_stats* st) {
    if (!p) return fail(TET_E_ARG, "null plan");
    return run(p->m, &p->g, proj, acc, 1, Op::BackwardF64, cuda_stream, st,
               p->has_opt ? &p->opt : nullptr, p);
}

tet_status tet_set_kernel_timing(tet_mesh_t m, int enable) {
    if (!m) return fail(TET_E_ARG, "null mesh");
    std::lock_guard<std::mutex> g(m->tmu);
    m->timing = enable != 0;
    return TET_OK;
}

tet_status tet_kernel_times(tet_mesh_t m, double ms[4], int64_t launches[4]) {
    if (!m || !ms || !launches) return fail(TET_E_ARG, "null argument");
    DeviceGuard guard(m->device);
    std::lock_guard<std::mutex> g(m->tmu);
    // busy time of each class = length of the UNION of its launch intervals:
    // a call's angle chunks run on two streams and may overlap (AuxStream)
    std::vector<std::pair<float, float>> iv[TET_K_COUNT];
    for (auto& r : m->pending) {
        float t0 = 0, t1 = 0;
        cudaError_t e = cudaEventElapsedTime(&t0, m->pending.front().a, r.a);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t1, m->pending.front().a, r.b);
        if (e != cudaSuccess) return cuda_fail(e, "tet_kernel_times (stream not synchronised?)");
        iv[r.kind].push_back({t0, t1});
        m->launches[r.kind] += 1;
    }
    for (auto& r : m->pending) {
        m->spare.push_back(r.a);
        m->spare.push_back(r.b);
    }
    m->pending.clear();
    for (int k = 0; k < TET_K_COUNT; ++k) {
        std::sort(iv[k].begin(), iv[k].end());
        double busy = 0, lo = 0, hi = 0;
        bool open = false;
        for (auto& x : iv[k]) {
            if (open && x.first <= hi) {
                hi = std::max(hi, (double)x.second);
                continue;
            }
            if (open) busy += hi - lo;
            lo = x.first;
            hi = x.second;
            open = true;
        }
        if (open) busy += hi - lo;
        m->ms[k] += busy;
    }
    for (int k = 0; k < TET_K_COUNT; ++k) {
        ms[k] = m->ms[k];
        launches[k] = m->launches[k];
        m->ms[k] = 0;
        m->launches[k] = 0;
    }
    return TET_OK;
}

tet_status tet_mesh_features(tet_mesh_t m, int64_t feat[4]) {
    if (!m || !feat) return fail(TET_E_ARG, "null argument");
    feat[0] = m->dev.tag16 ? 1 : 0;
    feat[1] = m->tag16_bytes;
    feat[2] = m->rtree_nodes;
    feat[3] = m->bvh_nodes;
    return TET_OK;
}

tet_status tet_mesh_info(tet_mesh_t m, int64_t info[8]) {
    if (!m || !info) return fail(TET_E_ARG, "null argument");
    info[0] = m->dev.nv;
    info[1] = m->dev.nt;
    info[2] = m->dev.nb;
    info[3] = m->device;
    info[4] = m->host.e;
    info[5] = m->bytes;
    info[6] = (int64_t)m->dev.l2_window_bytes;
    info[7] = m->host.reordered ? 1 : 0;
    return TET_OK;
}

}  // extern "C"
