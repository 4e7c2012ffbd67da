// extern "C" implementation of include/wrng_gpu.h.
//
// Host-side control for the engines (smem_impl.cuh, hbm_engine.cu,
// cluster_engine.cu), the counter mirror,
// host-output staging (generation overlapped with D2H copies), the optional
// host (glibc) initial pool, and state import/export in the reference's
// "WRNG" v1 format (serialize.cpp:6-13) plus our v2 for n = 4 / f32 / banks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace wg;

namespace {

struct Ctr {  // per-pool counter mirror (WallaceState, wallace.hpp:167-172)
    uint64_t pc = 0, avail = 0, emitted = 0;
    uint32_t active = 0;
};

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

// WRNG_GPU_NO_BULK=1 routes full-refill emission through warp stores (A/B
// measurements); the default is the bulk-copy engine.
const bool g_bulk_emit = std::getenv("WRNG_GPU_NO_BULK") == nullptr;
// Output alignment (bytes) of each bulk-copied span; the ragged ends leave
// through warp stores.  WRNG_GPU_BULK_ALIGN overrides it (A/B measurements).
uint32_t bulk_align_bytes() {
    const char* e = std::getenv("WRNG_GPU_BULK_ALIGN");
    const long v = e ? std::strtol(e, nullptr, 10) : 64;
    return v >= 16 && v <= 4096 && (v & (v - 1)) == 0 ? (uint32_t)v : 64u;
}
const uint32_t g_bulk_align = bulk_align_bytes();
// WRNG_GPU_CLUSTER=1 runs few-pool fills on the cluster engine (opt-in: its
// random DSMEM gathers are request-bound, slower than one CTA for C1;
// DESIGN.md §5).
const bool g_cluster = std::getenv("WRNG_GPU_CLUSTER") != nullptr;
// Small n = 4 pools (4x256, fp32 4x512) fill on the group engine, several
// pools per warp; WRNG_GPU_NO_GROUP=1 keeps them on one CTA per pool (A/B).
const bool g_group = std::getenv("WRNG_GPU_NO_GROUP") == nullptr;
// HBM engine: consecutive passes run as one persistent launch (k_hbm_run);
// WRNG_GPU_HBM_STEPWISE=1 launches one kernel per pass and per emission.
const bool g_hbm_run = std::getenv("WRNG_GPU_HBM_STEPWISE") == nullptr;
// WRNG_GPU_NO_WINDOW=1 sends small host fills through the device path too.
const bool g_no_window = std::getenv("WRNG_GPU_NO_WINDOW") != nullptr;

bool crossed(uint64_t before, uint64_t after, uint64_t period) {
    return period > 0 && after / period > before / period;  // wallace.cpp:182-184
}

// Host (glibc) uniform generator + Box-Muller, bit-identical to the
// reference's UniformState / box_muller_next (uniform.cpp:13-45,
// reference.cpp:9-22).  Used for the initial pool and for restarts of
// WRNG_GPU_INIT_HOST handles, so those stay bit-exact across restarts.
struct HostLfg {
    uint64_t t[kTable];
    uint32_t r = 0;
    uint64_t draws = 0;
    void seed(uint64_t seed, uint64_t stream) {  // uniform.cpp:23-32
        uint64_t s = seed ^ ((stream << 32) | (stream >> 32));
        for (uint32_t i = 0; i < kTable; ++i) {
            s += 0x9E3779B97F4A7C15ull;
            uint64_t z = s;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            t[i] = z ^ (z >> 31);
        }
        r = 0;
        for (uint32_t i = 0; i < kWarmup; ++i) word();
        draws = 0;
    }
    void load(const LfgState& l) {
        std::memcpy(t, l.table, sizeof(t));
        r = l.r;
        draws = l.draws;
    }
    void store(LfgState& l) const {
        std::memcpy(l.table, t, sizeof(t));
        l.r = r;
        l.draws = draws;
    }
    uint64_t word() {  // uniform.cpp:34-40
        uint32_t s = r + kGap;
        if (s >= kTable) s -= kTable;
        uint64_t w = t[r] + t[s];
        t[r] = w;
        if (++r == kTable) r = 0;
        return w;
    }
    double uniform() {  // uniform.cpp:42-45
        ++draws;
        return (double)(word() >> 11) * 0x1.0p-53;
    }
};

void host_box_muller(HostLfg& u, double& x, double& y) {  // reference.cpp:9-22
    double u1 = u.uniform();
    if (u1 == 0.0) u1 = 0x1.0p-53;
    double u2 = u.uniform();
    const double pi = 3.141592653589793;
    double radius = std::sqrt(-2.0 * std::log(u1));
    double angle = 2.0 * pi * u2;
    x = radius * std::cos(angle);
    y = radius * std::sin(angle);
}

// init_pool (wallace.cpp:158-167) of one pool into `vals` (natural order,
// n_arrays * N elements of the pool dtype): box_muller_fill of every array
// in order (N is even, so no partner is dropped), then withheld = the .x of
// one more pair, tracked = direct_sumsq (sequential, wallace.cpp:13-18).
void host_init_pool(HostLfg& u, uint64_t nvals, bool f64, char* vals, double& tracked,
                    double& withheld) {
    const double zero = 0.0;
    for (uint64_t i = 0; i < nvals; i += 2) {
        double x, y;
        host_box_muller(u, x, y);
        const double vx = zero + x, vy = zero + y;  // mu + sigma * z, mu = 0, sigma = 1
        if (f64) {
            reinterpret_cast<double*>(vals)[i] = vx;
            reinterpret_cast<double*>(vals)[i + 1] = vy;
        } else {
            reinterpret_cast<float*>(vals)[i] = (float)vx;
            reinterpret_cast<float*>(vals)[i + 1] = (float)vy;
        }
    }
    double wx, wy;
    host_box_muller(u, wx, wy);
    double q = 0.0;
    for (uint64_t i = 0; i < nvals; ++i) {
        const double d = f64 ? reinterpret_cast<double*>(vals)[i]
                             : (double)reinterpret_cast<float*>(vals)[i];
        q = q + d * d;
    }
    tracked = q;
    withheld = wx;
}

}  // namespace

struct wrng_gpu {
    wrng_gpu_config cfg{};
    uint32_t N = 0;
    uint64_t nvals = 0, cap = 0;
    size_t esize = 8;
    bool hbm = false;
    void* buf[2] = {nullptr, nullptr};
    PoolMeta* meta = nullptr;
    LfgState* lfg = nullptr;
    wrng_gpu_params* params = nullptr;  // device: per-pool param records / hbm batches
    size_t params_cap = 0;
    double* scratch = nullptr;
    unsigned long long* gbar = nullptr;  // HBM engine: k_hbm_run's grid barrier counter
    cudaStream_t stream = nullptr;       // internal stream
    cudaStream_t copy_stream = nullptr;  // D2H of staged host fills
    cudaStream_t last = nullptr;         // last stream work was queued on
    bool last_set = false;
    cudaEvent_t order_ev = nullptr;
    void* stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    cudaEvent_t gen_done[2] = {nullptr, nullptr}, copy_done[2] = {nullptr, nullptr};
    std::vector<Ctr> ctr;
    void* l2_base = nullptr;
    uint64_t l2_bytes = 0;
    float l2_hit = 0.f;
    uint64_t launches = 0;
    std::string err;
    // Host window (single-pool smem handles): small host-output fills are
    // served from a host copy of the exposed pool, so a caller filling a few
    // values at a time (the reference's own usage, e.g. acceptance.cpp:
    // 134-140) pays one device refill + one pool copy per refill, not a
    // device round trip per call.  `gen` counts device operations that may
    // change the pool; the window is valid while win_gen == gen.  Values the
    // host consumed leave the device counters stale (meta_dirty) until the
    // next device operation writes them (order_on).
    std::vector<char> win;
    uint64_t win_gen = ~0ull;
    uint64_t gen = 0;
    bool meta_dirty = false;
    // Small host-output fills (<= kSmallBytes): one device slab and a pinned
    // bounce buffer, one stream, one synchronisation (fill_host_small).
    void* small_dev = nullptr;
    void* small_host = nullptr;
    PoolMeta* meta_host = nullptr;  // pinned mirror for collect()
};

constexpr size_t kSmallBytes = (size_t)16 << 20;

namespace {

wrng_gpu_status fail(wrng_gpu* g, wrng_gpu_status s, const std::string& what) {
    if (g) g->err = what;
    return s;
}

wrng_gpu_status cuda_fail(wrng_gpu* g, cudaError_t e, const char* where) {
    return fail(g, WRNG_GPU_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// No C++ exception crosses the C ABI: host allocation failures map to
// ENOMEM, anything else to ECUDA.
template <class F>
wrng_gpu_status guarded(wrng_gpu* g, F&& f) {
    try {
        return f();
    } catch (const std::bad_alloc&) {
        return fail(g, WRNG_GPU_ENOMEM, "host allocation failed");
    } catch (...) {
        return fail(g, WRNG_GPU_ECUDA, "unexpected host exception");
    }
}

#define CK(expr)                                                   \
    do {                                                           \
        cudaError_t e_ = (expr);                                   \
        if (e_ != cudaSuccess) return cuda_fail(g, e_, #expr);     \
    } while (0)

#define LAUNCH(expr)                                               \
    do {                                                           \
        cudaError_t e_ = (expr);                                   \
        if (e_ != cudaSuccess) return cuda_fail(g, e_, #expr);     \
        ++g->launches;                                             \
    } while (0)

// HBM pools live in transposed storage (hbm_pos); every host boundary
// (read/write_pool, export/import, host init) sees natural order.
void permute_pool(const wrng_gpu* g, void* data, bool to_storage) {
    if (!g->hbm) return;
    const HbmSplit sp = hbm_split(g->N);
    if (sp.lc == 0) return;  // one row: identity
    const size_t es = g->esize;
    std::vector<char> tmp(g->nvals * es);
    char* d = static_cast<char*>(data);
    for (uint64_t i = 0; i < g->nvals; ++i) {
        const uint64_t pos = hbm_pos(i, g->N, sp);
        if (to_storage)
            std::memcpy(tmp.data() + pos * es, d + i * es, es);
        else
            std::memcpy(tmp.data() + i * es, d + pos * es, es);
    }
    std::memcpy(d, tmp.data(), tmp.size());
}

// Restarts of WRNG_GPU_INIT_HOST handles run glibc's Box-Muller on the host
// (the device libm differs from glibc by a few ulp), so the whole stream
// stays bit-identical to the reference's (wallace.cpp:236).
bool host_bm(const wrng_gpu* g) { return (g->cfg.flags & WRNG_GPU_INIT_HOST) != 0; }

// Orders work on stream `s` after everything queued so far on the handle.
// Every device operation goes through here: it invalidates the host window
// and first writes counters the host window advanced.
wrng_gpu_status order_on(wrng_gpu* g, cudaStream_t s) {
    ++g->gen;
    if (g->last_set && g->last != s) {
        CK(cudaEventRecord(g->order_ev, g->last));
        CK(cudaStreamWaitEvent(s, g->order_ev, 0));
    }
    g->last = s;
    g->last_set = true;
    if (g->meta_dirty) {
        for (uint32_t p = 0; p < g->cfg.pools; ++p) {
            const Ctr& c = g->ctr[p];
            LAUNCH(launch_hbm_setmeta(g->meta + p, c.pc, c.avail, c.emitted, c.active, s));
        }
        g->meta_dirty = false;
    }
    return WRNG_GPU_OK;
}

KernelArgs base_args(const wrng_gpu* g) {
    KernelArgs a{};
    a.buf[0] = g->buf[0];
    a.buf[1] = g->buf[1];
    a.meta = g->meta;
    a.lfg = g->lfg;
    a.N = g->N;
    a.f = g->cfg.throwaway_f;
    a.mode = g->cfg.scale_mode;
    a.pools = g->cfg.pools;
    a.restart = g->cfg.restart_interval_passes;
    a.drift = g->cfg.drift_check_period;
    a.seed = g->cfg.seed;
    a.stream0 = g->cfg.stream_id;
    a.mu = 0.0;
    a.sigma = 1.0;
    a.unit = 1;
    a.l2_base = g->l2_base;
    a.l2_bytes = g->l2_bytes;
    a.l2_hit = g->l2_hit;
    return a;
}

KernelArgs pool_args(const wrng_gpu* g, uint32_t p) {
    KernelArgs a = base_args(g);
    a.buf[0] = static_cast<char*>(g->buf[0]) + (size_t)p * g->nvals * g->esize;
    a.buf[1] = static_cast<char*>(g->buf[1]) + (size_t)p * g->nvals * g->esize;
    a.meta = g->meta + p;
    a.lfg = g->lfg + p;
    a.stream0 = g->cfg.stream_id + p;
    a.pools = 1;
    return a;
}

// ---- host (glibc) initial pool: bit-identical to init_pool --------------
wrng_gpu_status host_init(wrng_gpu* g) {
    const uint32_t P = g->cfg.pools;
    const size_t pbytes = g->nvals * g->esize;
    std::vector<char> vals(pbytes * P);  // the whole bank: one H2D copy
    std::vector<LfgState> lfg(P);
    std::vector<PoolMeta> meta(P);
    for (uint32_t p = 0; p < P; ++p) {
        HostLfg u;
        u.seed(g->cfg.seed, g->cfg.stream_id + p);
        char* v = vals.data() + (size_t)p * pbytes;
        meta[p] = PoolMeta{};
        host_init_pool(u, g->nvals, g->cfg.dtype == WRNG_GPU_F64, v, meta[p].tracked[0],
                       meta[p].withheld[0]);
        permute_pool(g, v, true);
        u.store(lfg[p]);
    }
    CK(cudaMemcpyAsync(g->buf[0], vals.data(), vals.size(), cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(g->lfg, lfg.data(), sizeof(LfgState) * P, cudaMemcpyHostToDevice,
                       g->stream));
    CK(cudaMemcpyAsync(g->meta, meta.data(), sizeof(PoolMeta) * P, cudaMemcpyHostToDevice,
                       g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return WRNG_GPU_OK;
}

// restart (wallace.cpp:236 -> init_pool) of the listed pools on the host,
// from each pool's current device uniform state: the pool in buffer `act`
// is replaced, tracked/withheld[act] set, avail = 0.  `m` is the host copy
// of the pools' meta (updated and written back); restart_pending := mark.
struct PoolAct {
    uint32_t p, act;
};
wrng_gpu_status host_restart(wrng_gpu* g, const std::vector<PoolAct>& which,
                             std::vector<PoolMeta>& m, uint32_t mark, cudaStream_t s) {
    CK(cudaStreamSynchronize(s));
    const size_t pbytes = g->nvals * g->esize;
    std::vector<char> vals(pbytes);
    for (const PoolAct& pa : which) {
        LfgState l;
        CK(cudaMemcpyAsync(&l, g->lfg + pa.p, sizeof(l), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        HostLfg u;
        u.load(l);
        PoolMeta& mm = m[pa.p];
        host_init_pool(u, g->nvals, g->cfg.dtype == WRNG_GPU_F64, vals.data(),
                       mm.tracked[pa.act], mm.withheld[pa.act]);
        permute_pool(g, vals.data(), true);
        u.store(l);
        mm.avail = 0;
        mm.restart_pending = mark;
        CK(cudaMemcpyAsync(static_cast<char*>(g->buf[pa.act]) + (size_t)pa.p * pbytes,
                           vals.data(), pbytes, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(g->lfg + pa.p, &l, sizeof(l), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(g->meta + pa.p, &mm, sizeof(mm), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // host buffers are reused
    }
    return WRNG_GPU_OK;
}

// After a smem launch with host_restart = 1: restart every pool that stopped
// at a restart (restart_pending == 1) on the host; a fill (`resume_fill`)
// then relaunches those pools from where they stopped, until none is left.
wrng_gpu_status finish_host_restarts(wrng_gpu* g, KernelArgs a, bool resume_fill,
                                     cudaStream_t s) {
    const uint32_t P = g->cfg.pools;
    std::vector<PoolMeta> m(P);
    for (;;) {
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpyAsync(m.data(), g->meta, sizeof(PoolMeta) * P, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<PoolAct> pend;
        for (uint32_t p = 0; p < P; ++p)
            if (m[p].restart_pending == 1 && !m[p].error) pend.push_back({p, m[p].active});
        if (pend.empty()) return WRNG_GPU_OK;
        wrng_gpu_status st = host_restart(g, pend, m, resume_fill ? 2u : 0u, s);
        if (st) return st;
        if (!resume_fill) return WRNG_GPU_OK;
        a.resume = 1;
        LAUNCH(launch_smem(g->cfg.n_arrays, g->cfg.dtype, a, s));
    }
}

// Pulls device meta; on any device-raised error, resynchronises the counter
// mirror from the device, clears the flags and reports the error.
wrng_gpu_status collect(wrng_gpu* g) {
    if (g->meta_dirty) {
        wrng_gpu_status st = order_on(g, g->stream);
        if (st) return st;
    }
    // the meta read is queued behind everything on the handle's streams and
    // lands in a pinned mirror: one synchronisation per stream
    const uint32_t P = g->cfg.pools;
    if (g->last_set && g->last != g->stream) {
        CK(cudaEventRecord(g->order_ev, g->last));
        CK(cudaStreamWaitEvent(g->stream, g->order_ev, 0));
    }
    CK(cudaStreamSynchronize(g->copy_stream));
    CK(cudaMemcpyAsync(g->meta_host, g->meta, sizeof(PoolMeta) * P, cudaMemcpyDeviceToHost,
                       g->stream));
    CK(cudaStreamSynchronize(g->stream));
    if (g->last_set && g->last != g->stream) CK(cudaStreamSynchronize(g->last));
    std::vector<PoolMeta> m(g->meta_host, g->meta_host + P);
    uint32_t code = 0;
    for (uint32_t p = 0; p < P; ++p) {
        if (m[p].error) {
            code = m[p].error;
            m[p].error = 0;
        }
    }
    if (!code) return WRNG_GPU_OK;
    for (uint32_t p = 0; p < P; ++p) {
        g->ctr[p].pc = m[p].pass_count;
        g->ctr[p].avail = m[p].avail;
        g->ctr[p].emitted = m[p].emitted;
        g->ctr[p].active = m[p].active;
    }
    CK(cudaMemcpy(g->meta, m.data(), sizeof(PoolMeta) * P, cudaMemcpyHostToDevice));
    return fail(g, (wrng_gpu_status)code,
                "corrupted_state_error: tracked sum of squares not positive, or the "
                "drift audit found the pool sum of squares off by more than 1e-3");
}

// ---- host-side plan (mirror of the smem kernel's control flow) -----------
struct Ev {
    enum Kind { EMIT, PASS, DRIFT, RESTART } kind;
    uint64_t pos = 0, take = 0, out_off = 0, emit_n = 0;
    uint32_t end_refill = 0;
};

// An audit inside a refill runs on the refill's counters (pass_count
// advanced, avail = cap, emitted not yet counted), so a failing audit leaves
// them where the reference's exception does (wallace.cpp:188-196).
Ev drift_event(const Ctr& c) {
    Ev e{Ev::DRIFT};
    e.pos = c.pc;
    e.take = c.avail;
    e.out_off = c.emitted;
    return e;
}

void plan_fill(const wrng_gpu* g, Ctr& c, uint64_t len, std::vector<Ev>* ev) {
    const uint64_t cap = g->cap, f = g->cfg.throwaway_f;
    const uint64_t R = g->cfg.restart_interval_passes, D = g->cfg.drift_check_period;
    uint64_t done = 0;
    if (c.avail > 0 && len > 0) {
        uint64_t take = std::min(len, c.avail);
        if (ev) {
            Ev e{Ev::EMIT};
            e.pos = cap - c.avail;
            e.take = take;
            e.out_off = 0;
            ev->push_back(e);
        }
        done = take;
        c.avail -= take;
    }
    if (!ev && R == 0 && done < len) {
        // no event list and no restarts: the counters in closed form (a bank
        // fill plans thousands of pools x thousands of refills per call)
        const uint64_t rem = len - done, nref = (rem + cap - 1) / cap;
        c.pc += nref * f;
        c.active ^= (uint32_t)((nref * f) & 1u);
        c.avail = cap - (rem - (nref - 1) * cap);
        c.emitted += len;
        return;
    }
    while (done < len) {
        const uint64_t before = c.pc;
        const bool will_restart = R > 0 && crossed(before, before + f, R);
        const uint64_t emit_n = will_restart ? 0 : std::min(len - done, cap);
        for (uint64_t i = 0; i < f; ++i) {
            if (ev) {
                Ev e{Ev::PASS};
                e.emit_n = i + 1 == f ? emit_n : 0;
                e.out_off = done;
                e.end_refill = i + 1 == f;
                ev->push_back(e);
            }
            ++c.pc;
            c.active ^= 1u;
        }
        c.avail = cap;
        if (crossed(before, c.pc, D) && ev) ev->push_back(drift_event(c));
        if (will_restart) {
            if (ev) ev->push_back(Ev{Ev::RESTART});
            c.avail = 0;
            continue;
        }
        done += emit_n;
        c.avail -= emit_n;
    }
    c.emitted += len;
}

void plan_refill(const wrng_gpu* g, Ctr& c, std::vector<Ev>* ev) {
    const uint64_t f = g->cfg.throwaway_f;
    const uint64_t before = c.pc;
    for (uint64_t i = 0; i < f; ++i) {
        if (ev) {
            Ev e{Ev::PASS};
            e.end_refill = i + 1 == f;
            ev->push_back(e);
        }
        ++c.pc;
        c.active ^= 1u;
    }
    c.avail = g->cap;
    if (crossed(before, c.pc, g->cfg.drift_check_period) && ev) ev->push_back(drift_event(c));
    if (g->cfg.restart_interval_passes > 0 &&
        crossed(before, c.pc, g->cfg.restart_interval_passes)) {
        if (ev) ev->push_back(Ev{Ev::RESTART});
        c.avail = 0;
    }
}

wrng_gpu_status ensure_params(wrng_gpu* g, size_t n) {
    if (n <= g->params_cap) return WRNG_GPU_OK;
    if (g->params) cudaFree(g->params);
    g->params = nullptr;
    size_t want = std::max<size_t>(n, 1024);
    CK(cudaMalloc(&g->params, want * sizeof(wrng_gpu_params)));
    g->params_cap = want;
    return WRNG_GPU_OK;
}

// Executes a plan on HBM pool p (host-driven: one launch per pass).
wrng_gpu_status run_hbm(wrng_gpu* g, uint32_t p, Ctr c, const std::vector<Ev>& ev,
                        KernelArgs a, cudaStream_t s) {
    const uint32_t NA = g->cfg.n_arrays, dt = g->cfg.dtype;
    size_t i = 0;
    while (i < ev.size()) {
        // batch the parameter draws of consecutive passes up to the next
        // audit or restart: a restart draws Box-Muller uniforms, and a
        // failing audit must leave the uniform state where the reference's
        // exception leaves it (no later pass drawn, wallace.cpp:188-196)
        size_t jend = i;
        while (jend < ev.size() && ev[jend].kind != Ev::RESTART && ev[jend].kind != Ev::DRIFT)
            ++jend;
        uint32_t npass = 0;
        for (size_t k = i; k < jend; ++k) npass += ev[k].kind == Ev::PASS;
        if (npass) {
            wrng_gpu_status st = ensure_params(g, npass);
            if (st) return st;
            LAUNCH(launch_hbm_params(NA, g->N, a.lfg, g->params, npass, a.meta, s));
        }
        uint32_t pi = 0;
        for (size_t k = i; k < jend; ++k) {
            const Ev& e = ev[k];
            if (e.kind == Ev::PASS && g_hbm_run) {
                // a run of consecutive passes: one persistent launch
                HbmRun run{};
                run.src0 = c.active;
                run.param0 = pi;
                while (k < jend && ev[k].kind == Ev::PASS && run.npass < kRunMax) {
                    const Ev& q = ev[k];
                    run.emit_n[run.npass] = q.emit_n;
                    run.out_off[run.npass] = q.out_off;
                    if (q.end_refill) run.end_mask |= 1ull << run.npass;
                    ++run.npass;
                    ++pi;
                    c.active ^= 1u;
                    ++k;
                }
                --k;
                cudaError_t re = launch_hbm_run(NA, dt, a, g->params, run, g->gbar, s);
                if (re == cudaErrorCooperativeLaunchTooLarge || re == cudaErrorNotSupported) {
                    // the device cannot co-schedule the grid (e.g. shared by
                    // another context): the same passes, one launch each
                    (void)cudaGetLastError();
                    for (uint32_t r = 0; r < run.npass; ++r) {
                        HbmPass ps{};
                        ps.src = run.src0 ^ (r & 1u);
                        ps.param_idx = run.param0 + r;
                        ps.emit_n = run.emit_n[r];
                        ps.out_off = run.out_off[r];
                        ps.end_refill = (uint32_t)((run.end_mask >> r) & 1u);
                        LAUNCH(launch_hbm_pass(NA, dt, a, g->params, ps, s));
                        if (ps.emit_n)
                            LAUNCH(launch_hbm_emit_t(NA, dt, a, ps.src ^ 1u, ps.emit_n,
                                                     ps.out_off, s));
                    }
                    continue;
                }
                LAUNCH(re);
                continue;
            }
            if (e.kind == Ev::EMIT) {
                LAUNCH(launch_hbm_emit(NA, dt, a, c.active, e.pos, e.take, e.out_off, s));
            } else if (e.kind == Ev::PASS) {
                HbmPass ps{};
                ps.src = c.active;
                ps.param_idx = pi++;
                ps.emit_n = e.emit_n;
                ps.out_off = e.out_off;
                ps.end_refill = e.end_refill;
                LAUNCH(launch_hbm_pass(NA, dt, a, g->params, ps, s));
                c.active ^= 1u;
                if (e.emit_n)
                    LAUNCH(launch_hbm_emit_t(NA, dt, a, c.active, e.emit_n, e.out_off, s));
            }
        }
        if (jend < ev.size() && ev[jend].kind == Ev::DRIFT) {
            const Ev& d = ev[jend];
            LAUNCH(launch_hbm_setmeta(a.meta, d.pos, d.take, d.out_off, c.active, s));
            LAUNCH(launch_hbm_drift(NA, dt, a, c.active, (g->cfg.flags & WRNG_GPU_DRIFT_TREE) != 0,
                                    g->scratch, s));
            ++jend;
        } else if (jend < ev.size()) {  // RESTART
            if (host_bm(g)) {
                std::vector<PoolMeta> m(g->cfg.pools);
                CK(cudaStreamSynchronize(s));
                CK(cudaMemcpyAsync(&m[p], a.meta, sizeof(PoolMeta), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                if (!m[p].error) {
                    wrng_gpu_status st = host_restart(g, {{p, c.active}}, m, 0u, s);
                    if (st) return st;
                }
            } else {
                LAUNCH(launch_hbm_init(NA, dt, a, c.active, 0, g->scratch, s));
            }
            ++jend;
        }
        i = jend;
    }
    return WRNG_GPU_OK;
}

// One device-output bank fill (no staging): `lay` places each pool's values.
wrng_gpu_status fill_device(wrng_gpu* g, void* out, int out_f32, const OutLayout& lay,
                            double mu, double sigma, cudaStream_t s, double* stats = nullptr) {
    const uint32_t P = g->cfg.pools;
    const bool unit = mu == 0.0 && sigma == 1.0;
    wrng_gpu_status st = order_on(g, s);
    if (st) return st;
    if (!g->hbm) {
        KernelArgs a = base_args(g);
        a.op = OP_FILL;
        a.out = out;
        a.out_f32 = out_f32;
        a.unit = unit;
        a.mu = mu;
        a.sigma = sigma;
        a.lay = lay;
        a.bulk_emit = g_bulk_emit && (reinterpret_cast<uintptr_t>(out) % (out_f32 ? 4 : 8)) == 0
                          ? g_bulk_align
                          : 0u;
        a.host_restart = host_bm(g) && g->cfg.restart_interval_passes > 0;
        a.stats = stats;
        const bool unit_same = unit && (out_f32 != 0) == (g->cfg.dtype == WRNG_GPU_F32);
        if (g_cluster && !stats && g->cfg.restart_interval_passes == 0 &&
            cluster_engine_fits(g->cfg.n_arrays, g->cfg.dtype, g->N, P))
            LAUNCH(launch_cluster(g->cfg.n_arrays, g->cfg.dtype, a, s));
        else if (g_group && !stats && unit_same && a.bulk_emit &&
                 g->cfg.restart_interval_passes == 0 &&
                 group_engine_fits(g->cfg.n_arrays, g->cfg.dtype, g->N, g->cfg.throwaway_f) &&
                 // its loop counters are 32-bit: passes per pool in this call
                 ((lay.len_base + 1) / g->cap + 2) * g->cfg.throwaway_f < (1ull << 31))
            LAUNCH(launch_group(g->cfg.dtype, a, s));
        else
            LAUNCH(launch_smem(g->cfg.n_arrays, g->cfg.dtype, a, s));
        if (a.host_restart) {
            st = finish_host_restarts(g, a, true, s);
            if (st) return st;
        }
        for (uint32_t p = 0; p < P; ++p)
            plan_fill(g, g->ctr[p], lay.len_base + (p < lay.len_extra ? 1 : 0), nullptr);
        return WRNG_GPU_OK;
    }
    const size_t esz = out_f32 ? 4 : 8;
    for (uint32_t p = 0; p < P; ++p) {
        const uint64_t len = lay.len_base + (p < lay.len_extra ? 1 : 0);
        if (len == 0) continue;
        const uint64_t off = (uint64_t)p * lay.off_stride + std::min<uint64_t>(p, lay.off_extra);
        KernelArgs a = pool_args(g, p);
        a.out = static_cast<char*>(out) + off * esz;
        a.out_f32 = out_f32;
        a.unit = unit;
        a.mu = mu;
        a.sigma = sigma;
        std::vector<Ev> ev;
        Ctr before = g->ctr[p];
        plan_fill(g, g->ctr[p], len, &ev);
        st = run_hbm(g, p, before, ev, a, s);
        if (st) return st;
        const Ctr& c = g->ctr[p];
        LAUNCH(launch_hbm_setmeta(a.meta, c.pc, c.avail, c.emitted, c.active, s));
    }
    return WRNG_GPU_OK;
}

wrng_gpu_status ensure_stage(wrng_gpu* g) {
    if (g->stage[0]) return WRNG_GPU_OK;
    g->stage_bytes = (size_t)256 << 20;
    for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&g->stage[b], g->stage_bytes));
        CK(cudaEventCreateWithFlags(&g->gen_done[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->copy_done[b], cudaEventDisableTiming));
        CK(cudaEventRecord(g->copy_done[b], g->copy_stream));
    }
    return WRNG_GPU_OK;
}

// Host-output fill: generation into two device slabs alternating with
// asynchronous D2H copies; pool p's segment stays contiguous in `out`.
wrng_gpu_status fill_host(wrng_gpu* g, void* out, int out_f32, uint64_t count, double mu,
                          double sigma, cudaStream_t s) {
    wrng_gpu_status st = ensure_stage(g);
    if (st) return st;
    const uint32_t P = g->cfg.pools;
    const size_t esz = out_f32 ? 4 : 8;
    const uint64_t base = count / P, extra = count % P;
    const uint64_t stage_elems = g->stage_bytes / esz;
    char* hout = static_cast<char*>(out);
    int b = 0;
    if (!g->hbm) {
        // Sub-chunk t covers stream positions [t, t + L) of every pool's
        // segment; the chunk that reaches the shorter segments' end is the
        // tail (pools p < extra hold one value more).
        const uint64_t L = std::max<uint64_t>(1, stage_elems / P);
        for (uint64_t t = 0;; t += L) {
            const bool tail = t + L > base;
            OutLayout lay{};
            lay.off_stride = L;
            lay.off_extra = 0;
            lay.len_base = tail ? base - t : L;
            lay.len_extra = tail ? extra : 0;
            const uint64_t wb = lay.len_base, we = lay.len_base + (tail ? 1 : 0);
            if (wb == 0 && (extra == 0 || !tail)) break;
            CK(cudaStreamWaitEvent(s, g->copy_done[b], 0));
            st = fill_device(g, g->stage[b], out_f32, lay, mu, sigma, s);
            if (st) return st;
            CK(cudaEventRecord(g->gen_done[b], s));
            CK(cudaStreamWaitEvent(g->copy_stream, g->gen_done[b], 0));
            if (extra > 0 && we > 0)  // pools [0, extra): segment pitch base + 1
                CK(cudaMemcpy2DAsync(hout + t * esz, (base + 1) * esz, g->stage[b], L * esz,
                                     we * esz, extra, cudaMemcpyDeviceToHost,
                                     g->copy_stream));
            if (P > extra && wb > 0)  // pools [extra, P): segment pitch base
                CK(cudaMemcpy2DAsync(hout + (extra * (base + 1) + t) * esz, base * esz,
                                     static_cast<char*>(g->stage[b]) + extra * L * esz,
                                     L * esz, wb * esz, P - extra, cudaMemcpyDeviceToHost,
                                     g->copy_stream));
            CK(cudaEventRecord(g->copy_done[b], g->copy_stream));
            b ^= 1;
            if (tail) break;
        }
    } else {
        for (uint32_t p = 0; p < P; ++p) {
            const uint64_t len = base + (p < extra ? 1 : 0);
            const uint64_t off = (uint64_t)p * base + std::min<uint64_t>(p, extra);
            for (uint64_t t = 0; t < len; t += stage_elems) {
                const uint64_t c = std::min<uint64_t>(stage_elems, len - t);
                CK(cudaStreamWaitEvent(s, g->copy_done[b], 0));
                // single-pool fill of c values into the slab
                KernelArgs a = pool_args(g, p);
                a.out = g->stage[b];
                a.out_f32 = out_f32;
                a.unit = mu == 0.0 && sigma == 1.0;
                a.mu = mu;
                a.sigma = sigma;
                st = order_on(g, s);
                if (st) return st;
                std::vector<Ev> ev;
                Ctr before = g->ctr[p];
                plan_fill(g, g->ctr[p], c, &ev);
                st = run_hbm(g, p, before, ev, a, s);
                if (st) return st;
                const Ctr& cc = g->ctr[p];
                LAUNCH(launch_hbm_setmeta(a.meta, cc.pc, cc.avail, cc.emitted, cc.active, s));
                CK(cudaEventRecord(g->gen_done[b], s));
                CK(cudaStreamWaitEvent(g->copy_stream, g->gen_done[b], 0));
                CK(cudaMemcpyAsync(hout + (off + t) * esz, g->stage[b], c * esz,
                                   cudaMemcpyDeviceToHost, g->copy_stream));
                CK(cudaEventRecord(g->copy_done[b], g->copy_stream));
                b ^= 1;
            }
        }
    }
    CK(cudaStreamSynchronize(g->copy_stream));
    return collect(g);
}

wrng_gpu_status run_op(wrng_gpu* g, Op op, wrng_gpu_params* params_host);

// Host-output fill of at most one refill's worth from the host window
// (fill, wallace.cpp:198-216): refills run on the device, each exposed pool
// is copied to the host once, and the values are emitted as mu + sigma * v
// in fp64 (rounded once for f32 output), the device emission's arithmetic.
wrng_gpu_status fill_window(wrng_gpu* g, void* out, int out_f32, uint64_t count, double mu,
                            double sigma) {
    Ctr& c = g->ctr[0];
    const bool f64 = g->esize == 8;
    uint64_t done = 0;
    while (done < count) {
        if (c.avail == 0) {
            wrng_gpu_status st = run_op(g, OP_REFILL, nullptr);
            if (st) return st;
            continue;  // a restart leaves avail = 0
        }
        if (g->win_gen != g->gen) {
            wrng_gpu_status st = collect(g);
            if (st) return st;
            g->win.resize(g->nvals * g->esize);
            CK(cudaMemcpyAsync(g->win.data(), g->buf[c.active], g->win.size(),
                               cudaMemcpyDeviceToHost, g->stream));
            CK(cudaStreamSynchronize(g->stream));
            g->win_gen = g->gen;
        }
        const uint64_t take = std::min(count - done, c.avail);
        const uint64_t pos = g->cap - c.avail;
        for (uint64_t i = 0; i < take; ++i) {
            const double v = f64 ? reinterpret_cast<const double*>(g->win.data())[pos + i]
                                 : (double)reinterpret_cast<const float*>(g->win.data())[pos + i];
            const double o = mu + sigma * v;
            if (out_f32)
                static_cast<float*>(out)[done + i] = (float)o;
            else
                static_cast<double*>(out)[done + i] = o;
        }
        done += take;
        c.avail -= take;
        g->meta_dirty = true;
    }
    c.emitted += count;
    g->meta_dirty = true;
    return WRNG_GPU_OK;
}

// Host-output fill that fits kSmallBytes: generate into one device slab,
// copy it to a pinned bounce buffer on the same stream, read the meta behind
// it, synchronise once, then copy to the caller's (possibly pageable) memory.
// The staged path's two slabs and copy stream only pay off for large fills.
wrng_gpu_status fill_host_small(wrng_gpu* g, void* out, int out_f32, uint64_t count, double mu,
                                double sigma) {
    if (!g->small_dev) {
        CK(cudaMalloc(&g->small_dev, kSmallBytes));
        CK(cudaMallocHost(&g->small_host, kSmallBytes));
    }
    const uint32_t P = g->cfg.pools;
    const size_t bytes = count * (out_f32 ? 4 : 8);
    OutLayout lay{count / P, count % P, count / P, count % P};
    wrng_gpu_status st = fill_device(g, g->small_dev, out_f32, lay, mu, sigma, g->stream);
    if (st) return st;
    CK(cudaMemcpyAsync(g->small_host, g->small_dev, bytes, cudaMemcpyDeviceToHost, g->stream));
    st = collect(g);
    if (st) return st;
    std::memcpy(out, g->small_host, bytes);
    return WRNG_GPU_OK;
}

wrng_gpu_status do_fill(wrng_gpu* g, void* out, int out_f32, uint64_t count, double mu,
                        double sigma, int out_is_device, void* stream) {
    if (!g) return WRNG_GPU_EINVAL;
    if (sigma < 0.0) return fail(g, WRNG_GPU_EINVAL, "fill: sigma must be >= 0");
    if (count > 0 && !out) return fail(g, WRNG_GPU_EINVAL, "fill: null output");
    DeviceGuard dg(g->cfg.device);
    if (count == 0) {
        for (auto& c : g->ctr) plan_fill(g, c, 0, nullptr);
        return WRNG_GPU_OK;
    }
    if (!out_is_device && g->cfg.pools == 1 && !g->hbm && count <= g->cap && !g_no_window)
        return fill_window(g, out, out_f32, count, mu, sigma);
    if (!out_is_device && count * (out_f32 ? 4 : 8) <= kSmallBytes && !stream)
        return fill_host_small(g, out, out_f32, count, mu, sigma);
    if (!out_is_device)
        return fill_host(g, out, out_f32, count, mu, sigma,
                         stream ? static_cast<cudaStream_t>(stream) : g->stream);
    // Device output: the caller's stream; NULL is the legacy default stream.
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t P = g->cfg.pools;
    OutLayout lay{count / P, count % P, count / P, count % P};
    return fill_device(g, out, out_f32, lay, mu, sigma, s);
}

// Runs an op on every pool (smem: one launch; hbm: per pool) and syncs.
wrng_gpu_status run_op(wrng_gpu* g, Op op, wrng_gpu_params* params_host) {
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = order_on(g, g->stream);
    if (st) return st;
    const uint32_t P = g->cfg.pools;
    if (op == OP_PASSES && params_host) {
        st = ensure_params(g, P);
        if (st) return st;
    }
    if (op == OP_RESTART && host_bm(g)) {  // restart() of a host-init handle
        st = collect(g);
        if (st) return st;
        std::vector<PoolMeta> m(P);
        CK(cudaMemcpyAsync(m.data(), g->meta, sizeof(PoolMeta) * P, cudaMemcpyDeviceToHost,
                           g->stream));
        std::vector<PoolAct> all;
        for (uint32_t p = 0; p < P; ++p) all.push_back({p, g->ctr[p].active});
        st = host_restart(g, all, m, 0u, g->stream);
        if (st) return st;
        for (uint32_t p = 0; p < P; ++p) g->ctr[p].avail = 0;
        return collect(g);
    }
    if (!g->hbm) {
        KernelArgs a = base_args(g);
        a.op = op;
        a.npasses = 1;
        a.params_out = (op == OP_PASSES && params_host) ? g->params : nullptr;
        a.host_restart = op == OP_REFILL && host_bm(g) && g->cfg.restart_interval_passes > 0;
        LAUNCH(launch_smem(g->cfg.n_arrays, g->cfg.dtype, a, g->stream));
        if (a.host_restart) {
            st = finish_host_restarts(g, a, false, g->stream);
            if (st) return st;
        }
        for (uint32_t p = 0; p < P; ++p) {
            Ctr& c = g->ctr[p];
            if (op == OP_PASSES) {
                ++c.pc;
                c.active ^= 1u;
                c.avail = 0;
            } else if (op == OP_REFILL) {
                plan_refill(g, c, nullptr);
            } else if (op == OP_RESTART) {
                c.avail = 0;
            }
        }
    } else {
        for (uint32_t p = 0; p < P; ++p) {
            KernelArgs a = pool_args(g, p);
            Ctr& c = g->ctr[p];
            if (op == OP_PASSES) {
                LAUNCH(launch_hbm_params(g->cfg.n_arrays, g->N, a.lfg, g->params + p, 1, a.meta,
                                         g->stream));
                HbmPass ps{};
                ps.src = c.active;
                ps.param_idx = 0;
                LAUNCH(launch_hbm_pass(g->cfg.n_arrays, g->cfg.dtype, a, g->params + p, ps,
                                       g->stream));
                ++c.pc;
                c.active ^= 1u;
                c.avail = 0;
            } else if (op == OP_REFILL) {
                std::vector<Ev> ev;
                Ctr before = c;
                plan_refill(g, c, &ev);
                st = run_hbm(g, p, before, ev, a, g->stream);
                if (st) return st;
                LAUNCH(launch_hbm_setmeta(a.meta, c.pc, c.avail, c.emitted, c.active, g->stream));
            } else if (op == OP_DRIFT) {
                LAUNCH(launch_hbm_drift(g->cfg.n_arrays, g->cfg.dtype, a, c.active,
                                        (g->cfg.flags & WRNG_GPU_DRIFT_TREE) != 0, g->scratch,
                                        g->stream));
            } else if (op == OP_RESTART) {
                LAUNCH(launch_hbm_init(g->cfg.n_arrays, g->cfg.dtype, a, c.active, 0, g->scratch,
                                       g->stream));
                c.avail = 0;
            }
        }
    }
    st = collect(g);
    if (op == OP_PASSES && params_host && st == WRNG_GPU_OK)
        CK(cudaMemcpy(params_host, g->params, sizeof(wrng_gpu_params) * P,
                      cudaMemcpyDeviceToHost));
    return st;
}

wrng_gpu_status validate(const wrng_gpu_config* c, bool check_restart) {
    if (c->pool_exponent < 8 || c->pool_exponent > 20) return WRNG_GPU_EINVAL;
    if (c->throwaway_f < 1) return WRNG_GPU_EINVAL;
    if (check_restart && c->restart_interval_passes > 0 &&
        c->restart_interval_passes <= c->throwaway_f)
        return WRNG_GPU_EINVAL;
    if (c->n_arrays != 2 && c->n_arrays != 4) return WRNG_GPU_EINVAL;
    if (c->dtype > 1 || c->scale_mode > 1 || c->pools < 1) return WRNG_GPU_EINVAL;
    return WRNG_GPU_OK;
}

// Allocates a handle without initialising pool contents.
wrng_gpu_status alloc_handle(const wrng_gpu_config* cfg, wrng_gpu** out) {
    wrng_gpu* g = new wrng_gpu;
    g->cfg = *cfg;
    g->N = 1u << cfg->pool_exponent;
    g->nvals = (uint64_t)cfg->n_arrays * g->N;
    g->cap = g->nvals - 1;
    g->esize = cfg->dtype == WRNG_GPU_F64 ? 8 : 4;
    g->hbm = (cfg->flags & WRNG_GPU_FORCE_HBM) || !smem_engine_fits(cfg->n_arrays, cfg->dtype, g->N);
    g->ctr.assign(cfg->pools, Ctr{});
    *out = g;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(g, WRNG_GPU_ENODEV, "no CUDA device");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(g, WRNG_GPU_ENODEV, "bad device");
    DeviceGuard dg(cfg->device);
    const size_t pool_bytes = (size_t)cfg->pools * g->nvals * g->esize;
    // both buffers in one allocation: one L2 access window covers them
    if (cudaMalloc(&g->buf[0], 2 * pool_bytes) != cudaSuccess)
        return fail(g, WRNG_GPU_ENOMEM, "pool allocation failed");
    g->buf[1] = static_cast<char*>(g->buf[0]) + pool_bytes;
    CK(cudaMemset(g->buf[0], 0, 2 * pool_bytes));
    // persisting-L2 window over both pool buffers: opt-in (WRNG_GPU_L2WIN=1);
    // measured 2 % slower on C2 (9.36 vs 9.17 ms/step)
    if (g->hbm && std::getenv("WRNG_GPU_L2WIN") != nullptr) {
        int maxp = 0, maxw = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, cfg->device);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, cfg->device);
        const size_t want = 2 * pool_bytes;
        if (maxp > 0 && maxw > 0) {
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t setaside = std::min<size_t>(want, (size_t)maxp);
            if (cur < setaside) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside);
            g->l2_base = g->buf[0];
            g->l2_bytes = std::min<size_t>(want, (size_t)maxw);
            g->l2_hit = (float)std::min(1.0, (double)setaside / (double)g->l2_bytes);
        }
    }
    CK(cudaMalloc(&g->meta, sizeof(PoolMeta) * cfg->pools));
    CK(cudaMallocHost(&g->meta_host, sizeof(PoolMeta) * cfg->pools));
    CK(cudaMemset(g->meta, 0, sizeof(PoolMeta) * cfg->pools));
    CK(cudaMalloc(&g->lfg, sizeof(LfgState) * cfg->pools));
    CK(cudaMalloc(&g->scratch, g->hbm ? hbm_drift_scratch_bytes(g->nvals) : sizeof(double) * 1024));
    if (g->hbm) {
        CK(cudaMalloc(&g->gbar, (kRunBarWords + kRunFlowWords) * sizeof(unsigned long long)));
    }
    CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g->order_ev, cudaEventDisableTiming));
    smem_engine_probe(g->stream);
    return WRNG_GPU_OK;
}

// ---- serialization helpers ----------------------------------------------
constexpr uint32_t kMagic = 0x57524E47;  // "WRNG" (serialize.cpp:20)

struct Writer {
    std::vector<uint8_t> b;
    void u8(uint8_t v) { b.push_back(v); }
    void u32(uint32_t v) {
        for (int i = 0; i < 4; ++i) b.push_back((uint8_t)(v >> (8 * i)));
    }
    void u64(uint64_t v) {
        for (int i = 0; i < 8; ++i) b.push_back((uint8_t)(v >> (8 * i)));
    }
    void f64(double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
    void raw(const void* p, size_t n) {
        const uint8_t* c = static_cast<const uint8_t*>(p);
        b.insert(b.end(), c, c + n);
    }
};

struct Reader {
    const uint8_t* p;
    size_t n, pos = 0;
    bool ok = true;
    bool take(size_t k) {
        if (!ok || n - pos < k) {
            ok = false;
            return false;
        }
        return true;
    }
    uint8_t u8() {
        if (!take(1)) return 0;
        return p[pos++];
    }
    uint32_t u32() {
        if (!take(4)) return 0;
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= (uint32_t)p[pos + i] << (8 * i);
        pos += 4;
        return v;
    }
    uint64_t u64() {
        if (!take(8)) return 0;
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
        pos += 8;
        return v;
    }
    double f64() {
        uint64_t u = u64();
        double d;
        std::memcpy(&d, &u, 8);
        return d;
    }
    bool raw(void* dst, size_t k) {  // dst == nullptr: skip k bytes
        if (!take(k)) return false;
        if (dst) std::memcpy(dst, p + pos, k);
        pos += k;
        return true;
    }
};

}  // namespace

extern "C" {

void wrng_gpu_config_default(wrng_gpu_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->pool_exponent = 10;
    c->throwaway_f = 3;
    c->scale_mode = WRNG_GPU_CHISQ;
    c->n_arrays = 2;
    c->restart_interval_passes = 0;
    c->drift_check_period = 64;
    c->seed = 0;
    c->stream_id = 0;
    c->dtype = WRNG_GPU_F64;
    c->pools = 1;
    c->device = 0;
    c->flags = 0;
}

static wrng_gpu_status create_impl(const wrng_gpu_config* cfg, wrng_gpu_t** out) {
    if (!cfg || !out) return WRNG_GPU_EINVAL;
    *out = nullptr;
    wrng_gpu_status st = validate(cfg, true);
    if (st) return st;
    wrng_gpu* g = nullptr;
    st = alloc_handle(cfg, &g);
    if (st) {
        wrng_gpu_destroy(g);
        return st;
    }
    DeviceGuard dg(cfg->device);
    if (cfg->flags & WRNG_GPU_INIT_HOST) {
        st = host_init(g);
    } else if (!g->hbm) {
        KernelArgs a = base_args(g);
        a.op = OP_INIT;
        cudaError_t e = launch_smem(cfg->n_arrays, cfg->dtype, a, g->stream);
        st = e == cudaSuccess ? WRNG_GPU_OK : cuda_fail(g, e, "init");
        ++g->launches;
    } else {
        for (uint32_t p = 0; p < cfg->pools && !st; ++p) {
            KernelArgs a = pool_args(g, p);
            cudaError_t e = launch_hbm_init(cfg->n_arrays, cfg->dtype, a, 0, 1, g->scratch, g->stream);
            st = e == cudaSuccess ? WRNG_GPU_OK : cuda_fail(g, e, "init");
            ++g->launches;
        }
    }
    if (!st) st = collect(g);
    if (st) {
        wrng_gpu_destroy(g);
        return st;
    }
    *out = g;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_create(const wrng_gpu_config* cfg, wrng_gpu_t** out) {
    return guarded(nullptr, [&] { return create_impl(cfg, out); });
}

void wrng_gpu_destroy(wrng_gpu_t* g) {
    if (!g) return;
    {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) == cudaSuccess && g->cfg.device >= 0 &&
            g->cfg.device < ndev) {
            DeviceGuard dg(g->cfg.device);
            if (g->stream) cudaStreamSynchronize(g->stream);
            if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);
            if (g->buf[0]) cudaFree(g->buf[0]);  // both buffers (one allocation)
            for (int b = 0; b < 2; ++b) {
                if (g->stage[b]) cudaFree(g->stage[b]);
                if (g->gen_done[b]) cudaEventDestroy(g->gen_done[b]);
                if (g->copy_done[b]) cudaEventDestroy(g->copy_done[b]);
            }
            if (g->meta) cudaFree(g->meta);
            if (g->meta_host) cudaFreeHost(g->meta_host);
            if (g->small_dev) cudaFree(g->small_dev);
            if (g->small_host) cudaFreeHost(g->small_host);
            if (g->lfg) cudaFree(g->lfg);
            if (g->params) cudaFree(g->params);
            if (g->scratch) cudaFree(g->scratch);
            if (g->gbar) cudaFree(g->gbar);
            if (g->order_ev) cudaEventDestroy(g->order_ev);
            if (g->stream) cudaStreamDestroy(g->stream);
            if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
        }
    }
    delete g;
}

wrng_gpu_status wrng_gpu_fill_f64(wrng_gpu_t* g, double* out, uint64_t count, double mu,
                                  double sigma, int out_is_device, void* stream) {
    return guarded(g, [&] { return do_fill(g, out, 0, count, mu, sigma, out_is_device, stream); });
}

wrng_gpu_status wrng_gpu_fill_f32(wrng_gpu_t* g, float* out, uint64_t count, double mu,
                                  double sigma, int out_is_device, void* stream) {
    return guarded(g, [&] { return do_fill(g, out, 1, count, mu, sigma, out_is_device, stream); });
}

wrng_gpu_status wrng_gpu_advance_pass(wrng_gpu_t* g, wrng_gpu_params* params) {
    if (!g) return WRNG_GPU_EINVAL;
    if (g->hbm && !params) {
        wrng_gpu_status st = ensure_params(g, g->cfg.pools);
        if (st) return st;
    }
    return guarded(g, [&] { return run_op(g, OP_PASSES, params); });
}

wrng_gpu_status wrng_gpu_refill(wrng_gpu_t* g) {
    if (!g) return WRNG_GPU_EINVAL;
    if (g->hbm) {
        wrng_gpu_status st = ensure_params(g, g->cfg.throwaway_f);
        if (st) return st;
    }
    return guarded(g, [&] { return run_op(g, OP_REFILL, nullptr); });
}

wrng_gpu_status wrng_gpu_drift_check(wrng_gpu_t* g) {
    if (!g) return WRNG_GPU_EINVAL;
    return guarded(g, [&] { return run_op(g, OP_DRIFT, nullptr); });
}

wrng_gpu_status wrng_gpu_restart(wrng_gpu_t* g) {
    if (!g) return WRNG_GPU_EINVAL;
    return guarded(g, [&] { return run_op(g, OP_RESTART, nullptr); });
}

wrng_gpu_status wrng_gpu_get_config(const wrng_gpu_t* g, wrng_gpu_config* out) {
    if (!g || !out) return WRNG_GPU_EINVAL;
    *out = g->cfg;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_get_counters(const wrng_gpu_t* g, uint32_t pool,
                                      wrng_gpu_counters* out) {
    if (!g || !out || pool >= g->cfg.pools) return WRNG_GPU_EINVAL;
    const Ctr& c = g->ctr[pool];
    out->pass_count = c.pc;
    out->numbers_emitted = c.emitted;
    out->avail = c.avail;
    out->active = c.active;
    out->pool_size = g->N;
    return WRNG_GPU_OK;
}

static wrng_gpu_status read_pool_impl(wrng_gpu_t* g, uint32_t pool, double* values,
                                   double* tracked, double* withheld) {
    if (!g || pool >= g->cfg.pools) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = collect(g);
    if (st) return st;
    PoolMeta m;
    CK(cudaMemcpy(&m, g->meta + pool, sizeof(m), cudaMemcpyDeviceToHost));
    const uint32_t act = m.active;
    if (values) {
        std::vector<char> raw(g->nvals * g->esize);
        CK(cudaMemcpy(raw.data(), static_cast<char*>(g->buf[act]) + (size_t)pool * raw.size(),
                      raw.size(), cudaMemcpyDeviceToHost));
        permute_pool(g, raw.data(), false);
        for (uint64_t i = 0; i < g->nvals; ++i)
            values[i] = g->esize == 8 ? reinterpret_cast<double*>(raw.data())[i]
                                      : (double)reinterpret_cast<float*>(raw.data())[i];
    }
    if (tracked) *tracked = m.tracked[act];
    if (withheld) *withheld = m.withheld[act];
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_read_pool(wrng_gpu_t* g, uint32_t pool, double* values,
                                   double* tracked, double* withheld) {
    return guarded(g, [&] { return read_pool_impl(g, pool, values, tracked, withheld); });
}

static wrng_gpu_status write_pool_impl(wrng_gpu_t* g, uint32_t pool, const double* values,
                                    double tracked, double withheld) {
    if (!g || pool >= g->cfg.pools) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = collect(g);
    if (st) return st;
    ++g->gen;  // the host window is stale
    PoolMeta m;
    CK(cudaMemcpy(&m, g->meta + pool, sizeof(m), cudaMemcpyDeviceToHost));
    const uint32_t act = m.active;
    if (values) {
        std::vector<char> raw(g->nvals * g->esize);
        for (uint64_t i = 0; i < g->nvals; ++i) {
            if (g->esize == 8)
                reinterpret_cast<double*>(raw.data())[i] = values[i];
            else
                reinterpret_cast<float*>(raw.data())[i] = (float)values[i];
        }
        permute_pool(g, raw.data(), true);
        CK(cudaMemcpy(static_cast<char*>(g->buf[act]) + (size_t)pool * raw.size(), raw.data(),
                      raw.size(), cudaMemcpyHostToDevice));
    }
    m.tracked[act] = tracked;
    m.withheld[act] = withheld;
    CK(cudaMemcpy(g->meta + pool, &m, sizeof(m), cudaMemcpyHostToDevice));
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_write_pool(wrng_gpu_t* g, uint32_t pool, const double* values,
                                    double tracked, double withheld) {
    return guarded(g, [&] { return write_pool_impl(g, pool, values, tracked, withheld); });
}

static wrng_gpu_status read_uniform_impl(wrng_gpu_t* g, uint32_t pool, uint64_t* table607,
                                      uint32_t* cursor_r, uint32_t* cursor_s,
                                      uint64_t* draws) {
    if (!g || pool >= g->cfg.pools) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = collect(g);
    if (st) return st;
    LfgState l;
    CK(cudaMemcpy(&l, g->lfg + pool, sizeof(l), cudaMemcpyDeviceToHost));
    if (table607) std::memcpy(table607, l.table, sizeof(l.table));
    if (cursor_r) *cursor_r = l.r;
    if (cursor_s) *cursor_s = (l.r + kGap) % kTable;
    if (draws) *draws = l.draws;
    return WRNG_GPU_OK;
}

static wrng_gpu_status write_uniform_impl(wrng_gpu_t* g, uint32_t pool, const uint64_t* table607,
                                          uint32_t cursor_r, uint32_t cursor_s, uint64_t draws) {
    if (!g || !table607 || pool >= g->cfg.pools) return WRNG_GPU_EINVAL;
    if (cursor_r >= kTable || (cursor_r + kGap) % kTable != cursor_s)
        return fail(g, WRNG_GPU_EINVAL, "write_uniform: cursors out of range");
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = collect(g);
    if (st) return st;
    ++g->gen;
    LfgState l;
    std::memcpy(l.table, table607, sizeof(l.table));
    l.r = cursor_r;
    l.pad_ = 0;
    l.draws = draws;
    CK(cudaMemcpyAsync(g->lfg + pool, &l, sizeof(l), cudaMemcpyHostToDevice, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_write_uniform(wrng_gpu_t* g, uint32_t pool, const uint64_t* table607,
                                       uint32_t cursor_r, uint32_t cursor_s, uint64_t draws) {
    return guarded(g, [&] {
        return write_uniform_impl(g, pool, table607, cursor_r, cursor_s, draws);
    });
}

wrng_gpu_status wrng_gpu_read_uniform(wrng_gpu_t* g, uint32_t pool, uint64_t* table607,
                                      uint32_t* cursor_r, uint32_t* cursor_s,
                                      uint64_t* draws) {
    return guarded(g, [&] { return read_uniform_impl(g, pool, table607, cursor_r, cursor_s, draws); });
}

static wrng_gpu_status export_state_impl(wrng_gpu_t* g, uint8_t* buf, size_t cap, size_t* size) {
    if (!g || !size) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = collect(g);
    if (st) return st;
    const uint32_t P = g->cfg.pools;
    std::vector<PoolMeta> m(P);
    std::vector<LfgState> l(P);
    CK(cudaMemcpy(m.data(), g->meta, sizeof(PoolMeta) * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(l.data(), g->lfg, sizeof(LfgState) * P, cudaMemcpyDeviceToHost));
    const size_t pbytes = g->nvals * g->esize;
    std::vector<uint8_t> vals[2];
    for (int b = 0; b < 2; ++b) {
        vals[b].resize(pbytes * P);
        CK(cudaMemcpy(vals[b].data(), g->buf[b], vals[b].size(), cudaMemcpyDeviceToHost));
        for (uint32_t p = 0; p < P; ++p) permute_pool(g, vals[b].data() + p * pbytes, false);
    }
    const bool v1 = g->cfg.n_arrays == 2 && g->cfg.dtype == WRNG_GPU_F64 && P == 1;
    Writer w;
    // header (serialize.cpp:82-96)
    w.u32(kMagic);
    w.u32(v1 ? 1 : 2);
    w.u32(g->cfg.pool_exponent);
    w.u32(g->cfg.throwaway_f);
    w.u8((uint8_t)g->cfg.scale_mode);
    w.u64(g->cfg.restart_interval_passes);
    w.u64(g->cfg.drift_check_period);
    w.u64(g->cfg.seed);
    w.u64(g->cfg.stream_id);
    if (!v1) {
        w.u32(g->cfg.n_arrays);
        w.u32(g->cfg.dtype);
        w.u32(P);
    }
    for (uint32_t p = 0; p < P; ++p) {
        const Ctr& c = g->ctr[p];
        w.u64(c.pc);
        w.u64(c.emitted);
        w.u64(c.avail);
        w.u8((uint8_t)c.active);
        for (uint32_t i = 0; i < kTable; ++i) w.u64(l[p].table[i]);  // (serialize.cpp:98-101)
        w.u32(l[p].r);
        w.u32((l[p].r + kGap) % kTable);
        w.u64(l[p].draws);
        for (int b = 0; b < 2; ++b) {  // both pools (serialize.cpp:103-110)
            const uint8_t* src = vals[b].data() + p * pbytes;
            if (v1) {
                const double* d = reinterpret_cast<const double*>(src);
                for (uint64_t i = 0; i < g->nvals; ++i) w.f64(d[i]);
            } else {
                w.raw(src, pbytes);  // little-endian IEEE bit patterns
            }
            w.f64(m[p].tracked[b]);
            w.f64(m[p].withheld[b]);
        }
    }
    *size = w.b.size();
    if (buf && cap >= w.b.size()) std::memcpy(buf, w.b.data(), w.b.size());
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_export_state(wrng_gpu_t* g, uint8_t* buf, size_t cap, size_t* size) {
    return guarded(g, [&] { return export_state_impl(g, buf, cap, size); });
}

static wrng_gpu_status import_state_impl(const uint8_t* bytes, size_t size, int32_t device,
                                      uint32_t flags, wrng_gpu_t** out) {
    if (!out || (!bytes && size)) return WRNG_GPU_EINVAL;
    *out = nullptr;
    Reader r{bytes, size};
    // load_state (serialize.cpp:115-169): magic, version, then fields with
    // range checks; truncation and trailing bytes are errors.
    uint32_t magic = r.u32();
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    if (magic != kMagic) return WRNG_GPU_EMALFORMED_BAD_MAGIC;
    uint32_t ver = r.u32();
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    if (ver != 1 && ver != 2) return WRNG_GPU_EMALFORMED_VERSION;
    wrng_gpu_config c;
    wrng_gpu_config_default(&c);
    c.device = device;
    c.flags = flags;  // INIT_HOST: this handle's restarts use the host Box-Muller
    c.pool_exponent = r.u32();
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    if (c.pool_exponent < 8 || c.pool_exponent > 20) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
    c.throwaway_f = r.u32();
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    if (c.throwaway_f < 1) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
    uint8_t mode = r.u8();
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    if (mode > 1) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
    c.scale_mode = mode;
    c.restart_interval_passes = r.u64();
    c.drift_check_period = r.u64();
    c.seed = r.u64();
    c.stream_id = r.u64();
    if (ver == 2) {
        c.n_arrays = r.u32();
        c.dtype = r.u32();
        c.pools = r.u32();
        if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
        if ((c.n_arrays != 2 && c.n_arrays != 4) || c.dtype > 1 || c.pools < 1 ||
            c.pools > (1u << 20))
            return WRNG_GPU_EMALFORMED_FIELD_RANGE;
    }
    if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
    const uint32_t N = 1u << c.pool_exponent;
    const uint64_t nvals = (uint64_t)c.n_arrays * N;
    const size_t esz = c.dtype == WRNG_GPU_F64 ? 8 : 4;
    const uint32_t P = c.pools;
    const size_t body = r.pos;
    // Two passes over the pool records.  The first reads only counters and
    // cursors, skipping the value bytes, so a malformed input is rejected in
    // the reference's field order before anything is allocated (a short
    // header must not size host buffers: the record sizes are fixed by the
    // header, the first pass proves the input holds them all).  The second,
    // on an input now known to be exactly P records long, copies the values.
    std::vector<Ctr> ctr;
    std::vector<LfgState> lfg;
    std::vector<PoolMeta> meta;
    std::vector<uint8_t> vals[2];
    for (int pass = 0; pass < 2; ++pass) {
        const bool store = pass == 1;
        r.pos = body;
        r.ok = true;
        if (store) {
            try {
                ctr.resize(P);
                lfg.resize(P);
                meta.resize(P);
                vals[0].resize(nvals * esz * P);
                vals[1].resize(nvals * esz * P);
            } catch (const std::bad_alloc&) {
                return WRNG_GPU_ENOMEM;
            }
        }
        for (uint32_t p = 0; p < P; ++p) {
            Ctr cc;
            LfgState ll;
            cc.pc = r.u64();
            cc.emitted = r.u64();
            cc.avail = r.u64();
            if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
            if (cc.avail > nvals - 1) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
            uint8_t act = r.u8();
            if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
            if (act > 1) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
            cc.active = act;
            for (uint32_t i = 0; i < kTable; ++i) ll.table[i] = r.u64();
            uint32_t cr = r.u32(), cs = r.u32();
            if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
            if (cr >= kTable || cs >= kTable) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
            if ((cs + kTable - cr) % kTable != kGap) return WRNG_GPU_EMALFORMED_FIELD_RANGE;
            ll.r = cr;
            ll.pad_ = 0;
            ll.draws = r.u64();
            PoolMeta mm{};
            for (int b = 0; b < 2; ++b) {
                uint8_t* dst = store ? vals[b].data() + (size_t)p * nvals * esz : nullptr;
                if (ver == 1) {
                    // v1 stores doubles; the value bytes are the LE bit patterns
                    r.raw(dst, nvals * 8);
                } else {
                    r.raw(dst, nvals * esz);
                }
                mm.tracked[b] = r.f64();
                mm.withheld[b] = r.f64();
            }
            if (!r.ok) return WRNG_GPU_EMALFORMED_TRUNCATED;
            if (store) {
                mm.pass_count = cc.pc;
                mm.avail = cc.avail;
                mm.emitted = cc.emitted;
                mm.active = cc.active;
                ctr[p] = cc;
                lfg[p] = ll;
                meta[p] = mm;
            }
        }
        if (r.pos != size) return WRNG_GPU_EMALFORMED_FIELD_RANGE;  // trailing bytes
    }
    wrng_gpu* g = nullptr;
    wrng_gpu_status st = alloc_handle(&c, &g);
    if (st) {
        wrng_gpu_destroy(g);
        return st;
    }
    DeviceGuard dg(device);
    g->ctr = ctr;
    for (int b = 0; b < 2; ++b) {
        for (uint32_t p = 0; p < P; ++p)
            permute_pool(g, vals[b].data() + (size_t)p * nvals * esz, true);
        cudaError_t e = cudaMemcpy(g->buf[b], vals[b].data(), vals[b].size(),
                                   cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            wrng_gpu_destroy(g);
            return WRNG_GPU_ECUDA;
        }
    }
    if (cudaMemcpy(g->lfg, lfg.data(), sizeof(LfgState) * P, cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(g->meta, meta.data(), sizeof(PoolMeta) * P, cudaMemcpyHostToDevice) !=
            cudaSuccess) {
        wrng_gpu_destroy(g);
        return WRNG_GPU_ECUDA;
    }
    *out = g;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_import_state(const uint8_t* bytes, size_t size, int32_t device,
                                      uint32_t flags, wrng_gpu_t** out) {
    return guarded(nullptr, [&] { return import_state_impl(bytes, size, device, flags, out); });
}

wrng_gpu_status wrng_gpu_synchronize(wrng_gpu_t* g) {
    if (!g) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    return collect(g);
}

const char* wrng_gpu_last_error(const wrng_gpu_t* g) { return g ? g->err.c_str() : ""; }

uint64_t wrng_gpu_kernel_launches(const wrng_gpu_t* g) { return g ? g->launches : 0; }

int64_t wrng_gpu_resident_pools(const wrng_gpu_config* cfg) {
    if (!cfg || validate(cfg, false) != WRNG_GPU_OK) return -(int64_t)WRNG_GPU_EINVAL;
    const uint32_t N = 1u << cfg->pool_exponent;
    if ((cfg->flags & WRNG_GPU_FORCE_HBM) || !smem_engine_fits(cfg->n_arrays, cfg->dtype, N))
        return 0;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || cfg->device < 0 ||
        cfg->device >= ndev)
        return -(int64_t)WRNG_GPU_ENODEV;
    DeviceGuard dg(cfg->device);
    smem_engine_probe(nullptr);
    int per_sm = 0, sms = 0;
    KernelArgs a{};
    a.op = OP_QUERY;
    a.N = N;
    a.f = cfg->throwaway_f;
    a.out = &per_sm;
    const bool grp = g_group && cfg->restart_interval_passes == 0 &&
                     group_engine_fits(cfg->n_arrays, cfg->dtype, N, cfg->throwaway_f);
    if ((grp ? launch_group(cfg->dtype, a, nullptr)
             : launch_smem(cfg->n_arrays, cfg->dtype, a, nullptr)) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess)
        return -(int64_t)WRNG_GPU_ECUDA;
    return (int64_t)per_sm * sms;
}

const char* wrng_gpu_engine(const wrng_gpu_t* g) { return g && g->hbm ? "hbm" : "smem"; }

static wrng_gpu_status moments_any(const void* dev, int is_f32, uint64_t n, double* out5,
                                   int32_t device, void* stream) {
    if (!dev || !out5 || n == 0) return WRNG_GPU_EINVAL;
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t nb = 148 * 8;
    double* part = nullptr;
    if (cudaMalloc(&part, sizeof(double) * (nb * 4 + 8)) != cudaSuccess) return WRNG_GPU_ENOMEM;
    cudaError_t e = launch_moments(dev, is_f32, n, part, nb, part + nb * 4, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess)
        e = cudaMemcpy(out5, part + nb * 4, sizeof(double) * 5, cudaMemcpyDeviceToHost);
    cudaFree(part);
    return e == cudaSuccess ? WRNG_GPU_OK : WRNG_GPU_ECUDA;
}

wrng_gpu_status wrng_gpu_moments_f32(const float* dev, uint64_t n, double* out5, int32_t device,
                                     void* stream) {
    return moments_any(dev, 1, n, out5, device, stream);
}

wrng_gpu_status wrng_gpu_moments_f64(const double* dev, uint64_t n, double* out5,
                                     int32_t device, void* stream) {
    return moments_any(dev, 0, n, out5, device, stream);
}

// ---- validation statistics -----------------------------
}  // extern "C"

namespace {

// chi2_sf (stats.cpp:40-87): regularized upper incomplete gamma, series /
// continued fraction split at x = a + 1.
double gamma_p_series(double a, double x) {
    double ap = a, term = 1.0 / a, sum = term;
    for (int i = 0; i < 100000; ++i) {
        ap += 1.0;
        term *= x / ap;
        sum += term;
        if (std::fabs(term) < std::fabs(sum) * 1e-16) break;
    }
    return sum * std::exp(-x + a * std::log(x) - std::lgamma(a));
}

double gamma_q_contfrac(double a, double x) {
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 100000; ++i) {
        const double an = -i * (i - a);
        b += 2.0;
        d = an * d + b;
        if (std::fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (std::fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (std::fabs(del - 1.0) < 1e-16) break;
    }
    return h * std::exp(-x + a * std::log(x) - std::lgamma(a));
}

// chi2_bins' statistic (stats.cpp:30-35): expected = total / k, bin order.
double chi2_statistic(const std::vector<uint64_t>& c, uint64_t total) {
    const double expected = (double)total / (double)c.size();
    double st = 0.0;
    for (uint64_t x : c) {
        const double d = (double)x - expected;
        st += d * d / expected;
    }
    return st;
}

// Device scratch of one statistics call.
struct StatBufs {
    wrng_gpu* g = nullptr;
    double* part = nullptr;           // per-block partials (4 per block)
    double* acc = nullptr;            // [0..3] moment sums, [4..7] lag sums
    unsigned long long* cnt = nullptr;  // [k] u, [k] v, [1] skipped
    void* tail[2] = {nullptr, nullptr};
    void* ad = nullptr;  // A^2 keys + sort scratch
    double* pst = nullptr;  // [pools][4] moment sums of the fused path
    static constexpr uint32_t kBlocks = 148 * 4;
    ~StatBufs() {
        cudaFree(ad);
        cudaFree(pst);
        cudaFree(part);
        cudaFree(acc);
        cudaFree(cnt);
        cudaFree(tail[0]);
        cudaFree(tail[1]);
    }
    cudaError_t init(uint32_t k, size_t tail_bytes, cudaStream_t s) {
        cudaError_t e = cudaMalloc(&part, sizeof(double) * 4 * kBlocks);
        if (e == cudaSuccess) e = cudaMalloc(&acc, sizeof(double) * 16);
        if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(unsigned long long) * (2 * k + 1));
        if (e == cudaSuccess && tail_bytes) e = cudaMalloc(&tail[0], tail_bytes);
        if (e == cudaSuccess && tail_bytes) e = cudaMalloc(&tail[1], tail_bytes);
        if (e == cudaSuccess) e = cudaMemsetAsync(acc, 0, sizeof(double) * 8, s);
        if (e == cudaSuccess)
            e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (2 * k + 1), s);
        return e;
    }
};

double autocorr_from_sums(const double* acc, uint64_t n, uint64_t pairs) {
    const double m = acc[0] / (double)n, P = (double)pairs;
    const double num = acc[4] - m * (acc[5] + acc[6]) + P * m * m;
    const double den = acc[7] - 2.0 * m * acc[5] + P * m * m;
    return den == 0.0 ? NAN : num / den;
}

}  // namespace

extern "C" {

double wrng_gpu_chi2_sf(double statistic, uint32_t dof) {
    if (statistic < 0.0 || dof < 1) return NAN;
    if (statistic == 0.0) return 1.0;
    const double a = 0.5 * dof, x = 0.5 * statistic;
    return x < a + 1.0 ? 1.0 - gamma_p_series(a, x) : gamma_q_contfrac(a, x);
}

wrng_gpu_status wrng_gpu_uv_counts(const void* dev, int32_t is_f32, uint64_t n, uint32_t k,
                                   uint64_t* counts_u, uint64_t* counts_v, uint64_t* skipped,
                                   int32_t device, void* stream) {
    if (!dev || !counts_u || !counts_v || k < 2 || k > 8192) return WRNG_GPU_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    StatBufs b;
    cudaError_t e = b.init(k, 0, s);
    if (e == cudaSuccess)
        e = launch_uv_counts(dev, is_f32, 1, n, n, k, b.cnt, b.cnt + k, b.cnt + 2 * k, s);
    std::vector<unsigned long long> h(2 * k + 1);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess)
        e = cudaMemcpy(h.data(), b.cnt, sizeof(unsigned long long) * h.size(),
                       cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return WRNG_GPU_ECUDA;
    for (uint32_t i = 0; i < k; ++i) {
        counts_u[i] = h[i];
        counts_v[i] = h[k + i];
    }
    if (skipped) *skipped = h[2 * k];
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_autocorr(const void* dev, int32_t is_f32, uint64_t n, uint64_t lag,
                                  double* r, int32_t device, void* stream) {
    if (!dev || !r || n < lag + 2) return WRNG_GPU_EINVAL;  // stats.cpp:112-113
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    StatBufs b;
    cudaError_t e = b.init(2, 0, s);
    if (e == cudaSuccess)
        e = launch_moment_sums(dev, is_f32, 1, n, n, b.part, StatBufs::kBlocks, b.acc, s);
    if (e == cudaSuccess)
        e = launch_ac_sums(dev, dev, is_f32, 1, n, n, lag, 0, b.part, StatBufs::kBlocks,
                           b.acc + 4, s);
    double acc[8];
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(acc, b.acc, sizeof(acc), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return WRNG_GPU_ECUDA;
    *r = autocorr_from_sums(acc, n, n - lag);
    return WRNG_GPU_OK;
}

static wrng_gpu_status validate_impl(wrng_gpu_t* g, uint64_t count, uint32_t k, uint64_t lag,
                                  uint32_t what, uint64_t* counts_u, uint64_t* counts_v,
                                  wrng_gpu_validation* out) {
    if (!g || !out || k < 2 || k > 8192) return WRNG_GPU_EINVAL;
    DeviceGuard dg(g->cfg.device);
    wrng_gpu_status st = ensure_stage(g);
    if (st) return st;
    const uint32_t P = g->cfg.pools;
    const int f32 = g->cfg.dtype == WRNG_GPU_F32;
    const size_t esz = f32 ? 4 : 8;
    const uint64_t base = count / P, extra = count % P;
    cudaStream_t s = g->stream;
    StatBufs b;
    CK(b.init(k, (size_t)P * lag * esz, s));
    const bool want_ad = (what & WRNG_GPU_VALIDATE_AD) != 0 && count > 0;
    if (want_ad) {
        if (cudaMalloc(&b.ad, ad_scratch_bytes(f32, count)) != cudaSuccess) {
            (void)cudaGetLastError();
            return fail(g, WRNG_GPU_ENOMEM, "validate: no device memory for the A^2 sort");
        }
    }
    uint64_t ad_at = 0;
    // smem engine: the moment sums are accumulated by the emitting passes
    // themselves (per pool, fixed order); the HBM engine reduces the slab
    const bool fused = !g->hbm;
    if (fused) {
        CK(cudaMalloc(&b.pst, sizeof(double) * 4 * P));
        CK(cudaMemsetAsync(b.pst, 0, sizeof(double) * 4 * P, s));
    }
    // windows of L values per pool (even: pairs never straddle windows), the
    // slab kept <= 64 MiB so the reductions re-read it from L2
    const uint64_t slab = std::min<uint64_t>(g->stage_bytes, (uint64_t)64 << 20) / esz;
    const uint64_t L = std::max<uint64_t>(2, (slab / P) & ~1ull);
    uint64_t have = 0;
    int cur = 0;
    for (uint64_t t = 0;; t += L) {
        const bool tail = t + L > base;
        OutLayout lay{};
        lay.off_stride = L;
        lay.len_base = tail ? base - t : L;
        lay.len_extra = tail ? extra : 0;
        if (lay.len_base == 0 && lay.len_extra == 0) break;
        st = fill_device(g, g->stage[0], f32, lay, 0.0, 1.0, s, fused ? b.pst : nullptr);
        if (st) return st;
        // groups of equal window length: [0, len_extra) one longer
        struct Grp {
            uint32_t p0, np;
            uint64_t len;
        } grp[2] = {{0, (uint32_t)lay.len_extra, lay.len_base + 1},
                    {(uint32_t)lay.len_extra, P - (uint32_t)lay.len_extra, lay.len_base}};
        for (const Grp& gr : grp) {
            if (gr.np == 0 || gr.len == 0) continue;
            const char* w = static_cast<const char*>(g->stage[0]) + (size_t)gr.p0 * L * esz;
            if (!fused)
                CK(launch_moment_sums(w, f32, gr.np, L, gr.len, b.part, StatBufs::kBlocks, b.acc,
                                      s));
            if (want_ad) {
                CK(ad_add_values(w, f32, gr.np, L, gr.len, b.ad, ad_at, s));
                ad_at += (uint64_t)gr.np * gr.len;
            }
            CK(launch_uv_counts(w, f32, gr.np, L, gr.len, k, b.cnt, b.cnt + k, b.cnt + 2 * k, s));
            if (lag) {
                const size_t to = (size_t)gr.p0 * lag * esz;
                const char* told = static_cast<const char*>(b.tail[cur]) + to;
                char* tnew = static_cast<char*>(b.tail[cur ^ 1]) + to;
                CK(launch_ac_sums(w, told, f32, gr.np, L, gr.len, lag, have, b.part,
                                  StatBufs::kBlocks, b.acc + 4, s));
                CK(launch_ac_tail(w, told, tnew, f32, gr.np, L, gr.len, lag, have, s));
            }
            g->launches += lag ? 6 : 4;
        }
        cur ^= 1;
        have = std::min<uint64_t>(lag, have + lay.len_base);
        if (tail) break;
    }
    double a2 = NAN;
    if (want_ad) {
        CK(ad_finish(f32, count, b.ad, b.acc + 8, s));
        g->launches += 2 + 5 * (f32 ? 4 : 8);
    }
    double acc[8];
    std::vector<unsigned long long> h(2 * k + 1);
    CK(cudaStreamSynchronize(s));
    if (want_ad) CK(cudaMemcpy(&a2, b.acc + 8, sizeof(double), cudaMemcpyDeviceToHost));
    if (fused) {  // pools in order
        std::vector<double> ps(4 * (size_t)P);
        CK(cudaMemcpy(ps.data(), b.pst, sizeof(double) * ps.size(), cudaMemcpyDeviceToHost));
        double sum[4] = {0.0, 0.0, 0.0, 0.0};
        for (uint32_t p = 0; p < P; ++p)
            for (int k = 0; k < 4; ++k) sum[k] += ps[4 * (size_t)p + k];
        CK(cudaMemcpy(b.acc, sum, sizeof(sum), cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(acc, b.acc, sizeof(acc), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.data(), b.cnt, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
    st = collect(g);
    if (st) return st;
    wrng_gpu_validation v{};
    v.n = count;
    const double dn = (double)count;
    v.m1 = acc[0] / dn;
    v.m2 = acc[1] / dn;
    v.m3 = acc[2] / dn;
    v.m4 = acc[3] / dn;
    v.z1 = v.m1 * std::sqrt(dn / 1.0);  // stats.cpp:103-105
    v.z2 = (v.m2 - 1.0) * std::sqrt(dn / 2.0);
    v.z4 = (v.m4 - 3.0) * std::sqrt(dn / 96.0);
    std::vector<uint64_t> cu(h.begin(), h.begin() + k), cv(h.begin() + k, h.begin() + 2 * k);
    for (uint64_t x : cu) v.uv_samples += x;
    v.uv_skipped = h[2 * k];
    v.k = k;
    v.dof = k - 1;
    if (v.uv_samples) {
        v.u_statistic = chi2_statistic(cu, v.uv_samples);
        v.v_statistic = chi2_statistic(cv, v.uv_samples);
        v.u_p = wrng_gpu_chi2_sf(v.u_statistic, v.dof);
        v.v_p = wrng_gpu_chi2_sf(v.v_statistic, v.dof);
    }
    v.lag = lag;
    uint64_t pairs = 0;
    for (uint32_t p = 0; p < P; ++p) {
        const uint64_t np = base + (p < extra ? 1 : 0);
        pairs += np > lag ? np - lag : 0;
    }
    v.autocorr = lag && pairs ? autocorr_from_sums(acc, count, pairs) : NAN;
    v.ad_a2 = a2;
    v.ad_n = want_ad ? count : 0;
    if (counts_u) std::copy(cu.begin(), cu.end(), counts_u);
    if (counts_v) std::copy(cv.begin(), cv.end(), counts_v);
    *out = v;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_validate(wrng_gpu_t* g, uint64_t count, uint32_t k, uint64_t lag,
                                  uint64_t* counts_u, uint64_t* counts_v,
                                  wrng_gpu_validation* out) {
    return guarded(g, [&] { return validate_impl(g, count, k, lag, 0, counts_u, counts_v, out); });
}

wrng_gpu_status wrng_gpu_validate_ex(wrng_gpu_t* g, uint64_t count, uint32_t k, uint64_t lag,
                                     uint32_t what, uint64_t* counts_u, uint64_t* counts_v,
                                     wrng_gpu_validation* out) {
    return guarded(g, [&] {
        return validate_impl(g, count, k, lag, what, counts_u, counts_v, out);
    });
}

wrng_gpu_status wrng_gpu_anderson_darling(const void* dev, int32_t is_f32, uint64_t n, double* a2,
                                          int32_t device, void* stream) {
    if (!dev || !a2 || n == 0) return WRNG_GPU_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* scratch = nullptr;
    if (cudaMalloc(&scratch, ad_scratch_bytes(is_f32 ? 1 : 0, n) + 64) != cudaSuccess) {
        (void)cudaGetLastError();
        return WRNG_GPU_ENOMEM;
    }
    double* res = reinterpret_cast<double*>(static_cast<char*>(scratch) +
                                            ad_scratch_bytes(is_f32 ? 1 : 0, n));
    cudaError_t e = ad_add_values(dev, is_f32 ? 1 : 0, 1, n, n, scratch, 0, s);
    if (e == cudaSuccess) e = ad_finish(is_f32 ? 1 : 0, n, scratch, res, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(a2, res, sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(scratch);
    return e == cudaSuccess ? WRNG_GPU_OK : WRNG_GPU_ECUDA;
}

wrng_gpu_status wrng_gpu_method_fill(int32_t method, uint64_t seed, uint64_t stream_id,
                                     uint32_t pools, void* dev_out, int32_t out_f32,
                                     uint64_t count, double mu, double sigma, int32_t f64_math,
                                     int32_t device, void* stream) {
    if ((method != 0 && method != 1) || pools == 0 || !(sigma >= 0.0) ||
        (count > 0 && !dev_out))
        return WRNG_GPU_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    if (count == 0) return WRNG_GPU_OK;
    DeviceGuard dg(device);
    const OutLayout lay{count / pools, count % pools, count / pools, count % pools};
    cudaError_t e = launch_method_fill(method, f64_math, seed, stream_id, pools, lay, mu, sigma,
                                       out_f32 ? 1u : 0u, dev_out,
                                       static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? WRNG_GPU_OK : WRNG_GPU_ECUDA;
}

wrng_gpu_status wrng_gpu_lfg_words(uint64_t seed, uint64_t stream_id, uint32_t pools,
                                   uint64_t count, uint64_t* host_out, int32_t device) {
    if (!host_out || pools == 0) return WRNG_GPU_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    DeviceGuard dg(device);
    uint64_t* d = nullptr;
    const size_t bytes = sizeof(uint64_t) * count * pools;
    if (cudaMalloc(&d, bytes ? bytes : 8) != cudaSuccess) return WRNG_GPU_ENOMEM;
    cudaError_t e = launch_lfg_words(seed, stream_id, pools, count, d, nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess && bytes) e = cudaMemcpy(host_out, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? WRNG_GPU_OK : WRNG_GPU_ECUDA;
}

}  // extern "C"
