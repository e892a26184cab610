// api.cu — context, host orchestration of Algorithm 1, and the C-ABI.
//
// The host side mirrors the reference's control flow (optimizer.cpp:36-220)
// and its RNG consumption order exactly; all arithmetic over splats, pixels
// and parameters runs in the kernels of project.cu, binning.cu, raster.cu,
// ssim.cu and update.cu.  There is no CPU fallback: without a CUDA device
// every entry point fails with SGTR_RUNTIME.
#include <dlfcn.h>

#include <algorithm>
#include <sstream>
#include <fstream>
#include <atomic>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

thread_local std::string g_last_error;

Error invalid(const std::string& m) { return Error(SGTR_INVALID_ARGUMENT, m); }
Error numeric(const std::string& m) { return Error(SGTR_NUMERIC, m); }

const char* const kGroupNames[5] = {"position", "scale", "rotation", "opacity", "color"};
int group_of(long long K, long long k) {  // scene.cpp:41-47
    if (k < 3 * K) return 0;
    if (k < 6 * K) return 1;
    if (k < 10 * K) return 2;
    if (k < 11 * K) return 3;
    return 4;
}

// ------------------------------------------------------------------ buffers
struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() {
        if (p) cudaFree(p);
    }
    void* ensure(size_t need) {
        if (need <= bytes && p) return p;
        if (p) SGTR_CUDA(cudaFree(p));
        p = nullptr;
        size_t nb = std::max(need, bytes + bytes / 4);
        nb = std::max<size_t>(nb, 256);
        SGTR_CUDA(cudaMalloc(&p, nb));
        bytes = nb;
        return p;
    }
    template <typename T>
    T* as(size_t n) {
        return static_cast<T*>(ensure(n * sizeof(T)));
    }
    template <typename T>
    T* get() const {
        return static_cast<T*>(p);
    }
};

// device status block (pinned host mirror in Ctx::hstat)
struct DevStatus {
    ViewStatus vs;
    int bad_index;
    int degenerate;
    double tr[5];
    double scalar;
    int queue_count;
    int n_large;
};

// std::mt19937_64, output for output (the reference's Rng wraps it,
// rng.hpp:15-72), with a block interface for the Hutchinson probes: the
// reference takes bit 0 of one output per coordinate, and bit 0 of a tempered
// output is the parity of (state word & kBit0) -- the tempering is linear
// over GF(2) -- so a probe's bits come straight from the twisted state,
// 312 words per twist, without the per-output tempering.
struct MT64 {
    static constexpr int N = 312, M = 156;
    static constexpr uint64_t kBit0 = 0x80080824000041ull;
    uint64_t mt[N];
    int idx = N;
    explicit MT64(uint64_t seed = 5489u) {
        mt[0] = seed;
        for (int i = 1; i < N; ++i)
            mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    void twist() {
        constexpr uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
        constexpr uint64_t A = 0xB5026F5AA96619E9ull;
        for (int i = 0; i < N - M; ++i) {
            const uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
            mt[i] = mt[i + M] ^ (x >> 1) ^ ((0 - (x & 1)) & A);
        }
        for (int i = N - M; i < N - 1; ++i) {
            const uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
            mt[i] = mt[i + M - N] ^ (x >> 1) ^ ((0 - (x & 1)) & A);
        }
        const uint64_t x = (mt[N - 1] & UM) | (mt[0] & LM);
        mt[N - 1] = mt[M - 1] ^ (x >> 1) ^ ((0 - (x & 1)) & A);
        idx = 0;
    }
    uint64_t operator()() {
        if (idx >= N) twist();
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        return y ^ (y >> 43);
    }
    // the standard text form of std::mt19937_64 (the state words, then the
    // position), so checkpoints stay readable by either
    friend std::ostream& operator<<(std::ostream& os, const MT64& g) {
        os << g.mt[0];
        for (int i = 1; i < N; ++i) os << ' ' << g.mt[i];
        return os << ' ' << g.idx;
    }
    friend std::istream& operator>>(std::istream& is, MT64& g) {
        for (int i = 0; i < N; ++i) is >> g.mt[i];
        return is >> g.idx;
    }
    // bit 0 of the next n outputs, packed LSB first into out[0 .. ceil(n/32))
    void low_bits(uint32_t* out, long long n) {
        long long w = 0, done = 0;
        uint32_t word = 0;
        int nb = 0;
        while (done < n) {
            if (idx >= N) twist();
            const int take = (int)std::min<long long>(N - idx, n - done);
            const uint64_t* p = mt + idx;
            for (int k = 0; k < take; ++k) {
                word |= (uint32_t)__builtin_parityll(p[k] & kBit0) << nb;
                if (++nb == 32) {
                    out[w++] = word;
                    word = 0;
                    nb = 0;
                }
            }
            idx += take;
            done += take;
        }
        if (nb) out[w] = word;
    }
};

// RNG with the reference's variate mappings (rng.hpp:15-72)
struct Rng {
    MT64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t s = 1) : gen(s) {}
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double log_uniform(double lo, double hi) {
        return std::exp(uniform(std::log(lo), std::log(hi)));
    }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare = r * std::sin(2.0 * M_PI * u2);
        have_spare = true;
        return r * std::cos(2.0 * M_PI * u2);
    }
    std::vector<int> sample(int n, int k) {
        std::vector<int> idx(n);
        for (int i = 0; i < n; ++i) idx[i] = i;
        const int m = std::min(k, n);
        for (int i = 0; i < m; ++i) {
            const int j = i + static_cast<int>(gen() % static_cast<uint64_t>(n - i));
            std::swap(idx[i], idx[j]);
        }
        idx.resize(m);
        return idx;
    }
};

// The draws of one Algorithm-1 step in the reference order
// (optimizer.cpp:193-211): |S1| sample, then on refresh steps the |S2|
// sample and nu probes of dim Rademacher draws, coordinate-ascending.
struct DrawKey {
    int M = 0;
    long long dim = 0;
    int b1 = 0, b2 = 0, nu = 0, l = 0;
    bool operator==(const DrawKey& o) const {
        return M == o.M && dim == o.dim && b1 == o.b1 && b2 == o.b2 && nu == o.nu && l == o.l;
    }
};

struct StepDraws {
    long long t = 0;
    std::vector<int> s1, s2;
    bool refresh = false;
    std::vector<uint32_t> bits;
    Rng after_s1;  // state to restore when the gradient phase fails
    Rng after;     // state after all of the step's draws
    // state after probe s (the reference draws each probe lazily,
    // optimizer.cpp:67-73, :86-87): restored when Hutchinson sample s fails
    std::vector<Rng> after_probe;
};

StepDraws draw_step(Rng& rng, long long t, const DrawKey& k, const std::atomic<bool>* stop) {
    StepDraws d;
    d.t = t;
    d.s1 = rng.sample(k.M, k.b1);
    d.after_s1 = rng;
    d.refresh = k.l <= 1 || t % k.l == 1;
    if (d.refresh) {
        d.s2 = rng.sample(k.M, k.b2);
        const long long words = (k.dim + 31) / 32;
        d.bits.assign(words * k.nu, 0u);
        for (int s = 0; s < k.nu; ++s) {
            uint32_t* w = d.bits.data() + words * s;
            constexpr long long kChunk = 1 << 20;  // bits between stop checks (a multiple of 32)
            for (long long base = 0; base < k.dim; base += kChunk) {
                if (stop && stop->load()) return d;
                rng.gen.low_bits(w + (base >> 5), std::min(kChunk, k.dim - base));
            }
            d.after_probe.push_back(rng);
        }
    }
    d.after = rng;
    return d;
}

// Runs the RNG ahead of the GPU on a host thread: the whole consumption
// schedule up to the next refresh step is known from the options, so the
// probes of the next refresh (dim draws each) are generated while the
// intervening steps run on the device.
struct Prefetcher {
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<StepDraws> q;
    bool done = true;
    std::atomic<bool> stop{false};
    DrawKey key;

    void start(const Rng& from, long long t_next, const DrawKey& k) {
        reset();
        key = k;
        done = false;
        stop = false;
        th = std::thread([this, from, t_next, k]() {
            Rng r = from;
            for (long long t = t_next; t < t_next + 64 && !stop.load(); ++t) {
                StepDraws d = draw_step(r, t, k, &stop);
                const bool last = d.refresh;
                {
                    std::lock_guard<std::mutex> g(mu);
                    q.push_back(std::move(d));
                }
                cv.notify_all();
                if (last) break;
            }
            {
                std::lock_guard<std::mutex> g(mu);
                done = true;
            }
            cv.notify_all();
        });
    }
    bool take(long long t, const DrawKey& k, StepDraws& out) {
        if (!th.joinable() || !(k == key)) return false;
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !q.empty() || done; });
        if (q.empty() || q.front().t != t) return false;
        out = std::move(q.front());
        q.pop_front();
        return true;
    }
    bool exhausted() {
        std::lock_guard<std::mutex> g(mu);
        return done && q.empty();
    }
    void reset() {
        stop = true;
        if (th.joinable()) th.join();
        q.clear();
        done = true;
        stop = false;
    }
    ~Prefetcher() { reset(); }
};

struct View {
    sgtr_camera cam;
    DevCam dc;
};

DevCam make_devcam(const sgtr_camera& c) {
    DevCam d;
    d.W = c.width;
    d.H = c.height;
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    if (!quat_rot(c.q_wc, d.w)) throw invalid("quat_to_rotation: degenerate quaternion");
    for (int i = 0; i < 3; ++i) d.t[i] = c.t_wc[i];
    for (int a = 0; a < 3; ++a)
        d.cen[a] = -(d.w[a] * c.t_wc[0] + d.w[3 + a] * c.t_wc[1] + d.w[6 + a] * c.t_wc[2]);
    return d;
}

// NCCL, loaded on demand so single-GPU use needs no NCCL at all
struct Nccl {
    void* lib = nullptr;
    int (*get_unique_id)(void*) = nullptr;
    int (*comm_init_rank)(void**, int, const char*, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    const char* (*get_error)(int) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    void load() {
        if (lib) return;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) throw Error(SGTR_RUNTIME, std::string("dlopen libnccl.so.2: ") + dlerror());
        get_unique_id = (int (*)(void*))dlsym(lib, "ncclGetUniqueId");
        all_reduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
            lib, "ncclAllReduce");
        get_error = (const char* (*)(int))dlsym(lib, "ncclGetErrorString");
        comm_destroy = (int (*)(void*))dlsym(lib, "ncclCommDestroy");
        all_gather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(
            lib, "ncclAllGather");
        if (!get_unique_id || !all_reduce)
            throw Error(SGTR_RUNTIME, "libnccl.so.2 lacks the required symbols");
    }
    void check(int rc, const char* what) {
        if (rc != 0)
            throw Error(SGTR_RUNTIME,
                        std::string(what) + ": " + (get_error ? get_error(rc) : "nccl error"));
    }
};
Nccl g_nccl;

// ncclCommInitRank takes ncclUniqueId (128 bytes) by value
struct UniqueId {
    char internal[128];
};
typedef int (*CommInitRankFn)(void**, int, UniqueId, int);

// Per-kernel-class CUDA-event timing (off unless bench.py asks for it):
// events bracket each launch on the context stream, durations are harvested
// after the stream synchronises.
enum KClass {
    KC_PROJECT, KC_DEPTH_SORT, KC_TILE_BIN, KC_RASTER_FWD, KC_SSIM, KC_GATHER,
    KC_RASTER_VJP, KC_CHAIN, KC_PROJECT_JVP, KC_RASTER_JVP, KC_TR_UPDATE, KC_TR_BISECT,
    KC_TR_APPLY, KC_TR_ROT, KC_COUNT
};
const char* const kClassNames[KC_COUNT] = {
    "project", "depth_sort_scan", "tile_binning", "raster_fwd", "ssim_residual",
    "ssim_gather", "raster_vjp", "chain", "project_jvp", "raster_jvp", "tr_update",
    "tr_bisect", "tr_apply", "tr_rotation"};

struct KTimer {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<int, size_t>> pending;  // class, index of start event
    double total_ms[KC_COUNT] = {};
    long long count[KC_COUNT] = {};
    ~KTimer() {
        for (auto e : pool) cudaEventDestroy(e);
    }
    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            SGTR_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    void harvest() {
        for (auto& p : pending) {
            float ms = 0.f;
            SGTR_CUDA(cudaEventElapsedTime(&ms, pool[p.second], pool[p.second + 1]));
            total_ms[p.first] += ms;
            count[p.first] += 1;
        }
        pending.clear();
        used = 0;
    }
};

}  // namespace

// in-process communicator (see allreduce below)
struct LoopGroup {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<double*> ptr;
    explicit LoopGroup(int n_) : n(n_), ptr(n_, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; }))
            throw Error(SGTR_RUNTIME, "loopback group: a rank did not reach the collective");
    }
};
struct Ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    long long launches = 0;
    KTimer timer;
    int K = 0;
    Buf x, x_alt, ghat, dhat, adam_m, adam_v, fused, applied, vecbuf;
    bool have_applied = false;
    std::vector<View> views;
    Buf gt;  // planar targets, one (3, H, W) block per view
    bool has_gt = false;
    Buf gtmom;  // per view [mu_b (3, H, W) | mbb (3, H, W)] of its target (SSIM windows)
    bool has_gtmom = false;
    // held-out views for evaluate_scene (any sizes; planar targets packed
    // back to back at eval_off[i])
    std::vector<View> eval_views;
    std::vector<long long> eval_off;
    Buf eval_gt, eval_sums;
    long long t = 0;
    Rng rng{1};       // committed state: all draws of completed steps
    Prefetcher prefetch;
    // per-view workspace
    Buf rec, trec, keys, keys_alt, keys32, keys32_alt, ids, ids_alt, rect, tcount, off_r;
    Buf tkeys, tkeys_alt, dval, dval_alt, dup_id, tile_start, tile_end, temp;
    Buf img, tfin, last, adj, tan, adjl1, Pf, Qf, Rf, partials, zbits, seam0, seam1, seam2;
    Buf dxbuf, etabuf, queue, tile_ids, inv, part, mask, tinfo, large, trect, off_id, ovals;
    DevStatus* dstat = nullptr;
    DevStatus* hstat = nullptr;  // pinned
    // further view lanes (stream + per-view workspace), swapped in by
    // use_lane so consecutive gradient views overlap: one view's projection,
    // sorts, binning and SSIM run beside another's raster passes
    static constexpr int kMaxLanes = 2;
    struct Lane {
        cudaStream_t st = nullptr;
        DevStatus* dstat = nullptr;
        DevStatus* hstat = nullptr;
#define SGTR_LANE_BUFS(X)                                                                    \
    X(rec) X(keys) X(keys_alt) X(keys32) X(keys32_alt) X(ids) X(ids_alt) X(rect) X(tcount)   \
    X(off_r) X(tkeys)                                                                        \
    X(tkeys_alt) X(dval) X(dval_alt) X(dup_id) X(tile_start) X(tile_end) X(temp)             \
    X(img) X(tfin) X(last) X(adj) X(adjl1) X(Pf) X(Qf) X(Rf) X(partials) X(tile_ids) X(inv) \
    X(part) X(mask) X(tinfo) X(large) X(trect) X(off_id) X(ovals)
#define SGTR_DECL(n) Buf n;
        SGTR_LANE_BUFS(SGTR_DECL)
#undef SGTR_DECL
    } spare[kMaxLanes - 1];
    int cur_lane = 0;
    int slot_of[kMaxLanes] = {-1, 0};  // where each lane's workspace sits (-1: active)
    Buf gacc[kMaxLanes];         // gacc[1]: the second gradient accumulator (odd local views)
    cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes] = {};
    double* htail = nullptr;     // pinned staging for the fused tail
    size_t htail_n = 0;
    int nranks = 1, rank = 0;
    int refresh_bands = 1;  // bands per rank of each refresh view (sgtr_set_refresh_bands)
    int tr_shards = 1;      // radius shards run back to back on one rank (sgtr_set_tr_shards)
    int fail_sample = -1;   // Hutchinson sample of the last step's failure (sgtr_step_failed_sample)
    long long dup_cap = 0;  // capacity of the per-view duplicate arrays (grows, never shrinks)
    Buf stage;              // shard-major staging for the radius all-gather
    void* comm = nullptr;
    LoopGroup* loop = nullptr;  // in-process communicator (sgtr_comm_init_loopback)
    Buf loopbuf;
    bool collective() const { return (comm || loop) && nranks > 1; }

    ~Ctx() {
        prefetch.reset();
        if (comm && g_nccl.comm_destroy) {
            cudaSetDevice(device);
            cudaStreamSynchronize(st);
            g_nccl.comm_destroy(comm);
        }
        if (dstat) cudaFree(dstat);
        if (hstat) cudaFreeHost(hstat);
        if (st) cudaStreamDestroy(st);
        for (Lane& l : spare) {
            if (l.dstat) cudaFree(l.dstat);
            if (l.hstat) cudaFreeHost(l.hstat);
            if (l.st) cudaStreamDestroy(l.st);
        }
        if (htail) cudaFreeHost(htail);
        if (ev_fork) cudaEventDestroy(ev_fork);
        for (cudaEvent_t e : ev_join)
            if (e) cudaEventDestroy(e);
    }
    int nb = 0;  // SH coefficients per channel beyond DC ((d+1)^2 - 1; extension)
    long long dim() const { return (14LL + 3LL * nb) * K; }
    double* X() const { return x.get<double>(); }
};

namespace {

struct ViewRender {
    int W, H;
    int n_visible;   // -1 on a deferred view (not read back)
    long long n_dup;  // -1 on a deferred view
    long long cap;    // capacity of the duplicate arrays the view used
    TileLists tl;
    int err_kind;  // 0 none, 1 non-finite parameter, 2 degenerate quaternion
    int err_index;
};

// where a deferred view (render_view without a host round trip) reports its
// error, duplicate total and capacity overflow: slots of the step's fused
// tail (errk/erri/ndup may be null: another rank or band reports them)
struct ViewSlots {
    double *errk = nullptr, *erri = nullptr, *ndup = nullptr, *ovf = nullptr;
};

void bind(Ctx& c) { SGTR_CUDA(cudaSetDevice(c.device)); }

// make lane L the context's current stream + per-view workspace
void use_lane(Ctx& c, int L) {
    if (L == c.cur_lane) return;
    const int slot = c.slot_of[L];
    Ctx::Lane& sp = c.spare[slot];
    std::swap(c.st, sp.st);
    std::swap(c.dstat, sp.dstat);
    std::swap(c.hstat, sp.hstat);
#define SGTR_SWAP(n)                \
    std::swap(c.n.p, sp.n.p);       \
    std::swap(c.n.bytes, sp.n.bytes);
    SGTR_LANE_BUFS(SGTR_SWAP)
#undef SGTR_SWAP
    c.slot_of[c.cur_lane] = slot;
    c.slot_of[L] = -1;
    c.cur_lane = L;
}

// stream of lane L whether or not it is the active one
cudaStream_t lane_stream(Ctx& c, int L) {
    return L == c.cur_lane ? c.st : c.spare[c.slot_of[L]].st;
}

int lanes_knob() {
    const char* v = getenv("SGTR_LANES");
    return v ? std::max(1, std::min(2, atoi(v))) : 2;  // (1 disables the overlap)
}

struct Timed {
    Ctx& c;
    int cls;
    size_t idx = 0;
    Timed(Ctx& ctx, int k) : c(ctx), cls(k) {
        if (!c.timer.on) return;
        if (c.timer.used % 2) c.timer.used++;  // keep start/stop pairs adjacent
        idx = c.timer.used;
        SGTR_CUDA(cudaEventRecord(c.timer.next(), c.st));
    }
    ~Timed() {
        if (!c.timer.on) return;
        cudaEventRecord(c.timer.next(), c.st);
        c.timer.pending.push_back({cls, idx});
    }
};

// NVTX range over a scope (header-only NVTX 3: a no-op unless a profiler
// injects itself), so nsys / ncu timelines show the step's phases
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

void harvest_timing(Ctx& c) {
    if (c.timer.on) c.timer.harvest();
}

double* img_ptr(Ctx& c, Buf& b, int P) { return b.as<double>(3LL * P); }

// capacity for `need` duplicates.  Every view sorts `cap` tile keys (the
// tail padded), so the headroom is small: 1/16, enough that the views of later
// steps (the same scene, slowly changing) rarely outgrow it
long long grow_cap(long long need) { return need + need / 16 + 4096; }

// K1..K7 for one camera on the context's scene
// row0/row1: the tile rows the forward raster covers (a refresh band plus
// its halo); row1 < 0 renders the whole view.
// Without `defer`, the view's status and duplicate total are read back after
// the depth sort (one host round trip: errors are returned or thrown, the
// duplicate arrays sized exactly).  With `defer` nothing is read back: the
// duplicate arrays keep the context's capacity, and the status, the total and
// an overflow count go to the step's tail slots (k_view_end), checked once
// per step; an overflowing view renders nothing and the step is rerun.
ViewRender render_view(Ctx& c, const DevCam& dc, const RenderP& ro, bool throw_errors,
                       int row0 = 0, int row1 = -1, const ViewSlots* defer = nullptr) {
    ViewRender vr{};
    vr.W = dc.W;
    vr.H = dc.H;
    const int K = c.K;
    const int tiles_x = ceil_div(dc.W, kTile), tiles_y = ceil_div(dc.H, kTile);
    const int n_tiles = tiles_x * tiles_y;
    BinBuffers b;
    b.keys = c.keys.as<unsigned long long>(K + 1);
    b.keys_alt = c.keys_alt.as<unsigned long long>(K + 1);
    b.keys32 = c.keys32.as<unsigned int>(K + 1);
    b.keys32_alt = c.keys32_alt.as<unsigned int>(K + 1);
    b.ids = c.ids.as<int>(K + 1);
    b.ids_alt = c.ids_alt.as<int>(K + 1);
    b.rect = c.rect.as<int4>(K + 1);
    b.tcount = c.tcount.as<int>(K + 1);
    b.tinfo = c.tinfo.as<int4>(K + 1);
    b.large = c.large.as<int>(K + 1);
    b.n_large = &c.dstat->n_large;
    b.off_r = c.off_r.as<long long>(K + 1);
    b.off_id = c.off_id.as<long long>(std::max(K, 1));
    b.tile_start = c.tile_start.as<int>(std::max(n_tiles, 1));
    b.tile_end = c.tile_end.as<int>(std::max(n_tiles, 1));
    b.temp = c.temp.ensure(std::max(depth_sort_temp_bytes(K), scan_temp_bytes(K)));
    b.temp_bytes = c.temp.bytes;
    double* rec = c.rec.as<double>((size_t)kRec * (K + 1));
    b.rec = rec;
    if (c.dup_cap == 0) c.dup_cap = 2LL * K + 4096;  // grown on demand (the tile sort runs on it)

    view_begin(c.st, &c.dstat->vs);
    {
        Timed t(c, KC_PROJECT);
        launch_project(c.st, c.X(), K, c.nb, dc, ro, rec, b.keys, b.keys32, b.ids, b.rect,
                       b.tcount, b.tinfo, &c.dstat->vs);
    }
    {
        Timed t(c, KC_DEPTH_SORT);
        depth_sort_and_scan(c.st, b, K);
    }
    // view begin, project, onesweep sort (histogram + 5 passes), tie fix, scan (init + scan)
    c.launches += 1 + 1 + 6 + 1 + 2;
    if (defer) {
        view_end(c.st, &c.dstat->vs, b.off_r + K, c.dup_cap, defer->errk, defer->erri,
                 defer->ndup, defer->ovf);
        c.launches += 1;
        vr.n_visible = -1;
        vr.n_dup = -1;
    } else {
        SGTR_CUDA(cudaMemcpyAsync(&c.hstat->vs, &c.dstat->vs, sizeof(ViewStatus),
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaMemcpyAsync(&c.hstat->vs.n_dup, b.off_r + K, sizeof(long long),
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        const ViewStatus vs = c.hstat->vs;
        if (vs.nonfinite_splat != INT_MAX) {
            vr.err_kind = 1;
            vr.err_index = vs.nonfinite_splat;
        } else if (vs.degenerate_splat != INT_MAX) {
            vr.err_kind = 2;
            vr.err_index = vs.degenerate_splat;
        }
        if (vr.err_kind && throw_errors) {
            if (vr.err_kind == 1)
                throw numeric("rasterize: non-finite parameter in splat " +
                              std::to_string(vr.err_index));
            throw invalid("quat_to_rotation: degenerate quaternion");
        }
        if (vr.err_kind) return vr;
        vr.n_visible = vs.n_visible;
        vr.n_dup = vs.n_dup;
        if (vr.n_dup > INT_MAX) throw Error(SGTR_RUNTIME, "binning: more than 2^31 tile duplicates");
        if (vr.n_dup > c.dup_cap) c.dup_cap = grow_cap(vr.n_dup);
    }
    const long long cap = c.dup_cap;
    vr.cap = cap;
    b.tkeys = c.tkeys.as<unsigned int>(cap);
    b.tkeys_alt = c.tkeys_alt.as<unsigned int>(cap);
    b.dval = c.dval.as<int>(cap);
    b.dval_alt = c.dval_alt.as<int>(cap);
    b.dup_id = c.dup_id.as<int>(cap);
    b.tile_ids = c.tile_ids.as<int>(cap);
    b.trect = c.trect.as<int4>(cap);
    b.temp = c.temp.ensure(std::max({depth_sort_temp_bytes(K), scan_temp_bytes(K),
                                     tile_sort_temp_bytes(cap, n_tiles)}));
    b.temp_bytes = c.temp.bytes;
    {
        Timed t(c, KC_TILE_BIN);
        bin_tiles(c.st, b, K, tiles_x, n_tiles, cap);
    }
    c.launches += 6;  // emit (2), padding, tile sort (histogram + 2 passes), ranges + ids
    vr.tl = TileLists{tiles_x, tiles_y, b.tile_start, b.tile_end, b.dval_alt,
                      b.dup_id,  b.tile_ids, b.trect, row0,
                      row1 < 0 ? tiles_y : row1};
    // the raster kernels' CTAs in order of decreasing tile-list length: the
    // long tiles start first, so the grid does not end on a few of them
    // (SGTR_TILE_ORDER=0: row-major); full frames only
    static const bool by_length = getenv("SGTR_TILE_ORDER") ? atoi(getenv("SGTR_TILE_ORDER")) : 1;
    if (by_length && vr.tl.row0 == 0 && vr.tl.row1 == tiles_y) {
        Timed t(c, KC_TILE_BIN);
        int* order = c.ovals.as<int>(n_tiles);
        launch_tile_order(c.st, b.tile_start, b.tile_end, n_tiles, order);
        vr.tl.order = order;
        c.launches += 1;
    }
    const int P = dc.W * dc.H;
    Timed t(c, KC_RASTER_FWD);
    launch_raster_fwd(c.st, vr.tl, rec, dc.W, dc.H, ro, img_ptr(c, c.img, P),
                      c.tfin.as<double>(P), c.last.as<int>(P));
    c.launches += 1;
    return vr;
}

// K10 + K11 for an image-space adjoint already in c.adj
void backward_view(Ctx& c, const DevCam& dc, const RenderP& ro, const ViewRender& vr, int mode,
                   const double* zdense, const uint32_t* zbits, double* acc, double* flag) {
    const long long nd = std::max(vr.cap, 1LL);
    double* part = c.part.as<double>((size_t)kVjpSlots * kPartStride * nd);
    unsigned char* mask = c.mask.as<unsigned char>((size_t)kVjpSlots * nd);
    {
        Timed t(c, KC_RASTER_VJP);
        SGTR_CUDA(cudaMemsetAsync(mask, 0, (size_t)kVjpSlots * nd, c.st));
        launch_raster_vjp_warp(c.st, vr.tl, c.rec.get<double>(), vr.W, vr.H, ro,
                               c.adj.get<double>(), c.tfin.get<double>(), c.last.get<int>(), part,
                               mask);
    }
    Timed t(c, KC_CHAIN);
    const long long* off_id = c.off_id.get<long long>();  // written by K4 (bin_tiles)
    const int slots = vjp_slots(vr.tl.tiles_x * (vr.tl.row1 - vr.tl.row0));
    launch_chain_warp(c.st, mode, c.X(), c.K, c.nb, dc, ro, off_id, c.tcount.get<int>(), vr.cap,
                      slots, part, mask, zdense, zbits, acc, flag);
    c.launches += 2;
}

struct SsimOut {
    double* adjl1;
};

// K8/K13 + K9: residual chain adjoint of the rendered image into c.adj
// by0/by1: SSIM block rows to evaluate, gy0/gy1: block rows of the gathered
// adjoint (a refresh band: the band's rows, SSIM on the band +- one block)
void residual_adjoint(Ctx& c, int mode, int W, int H, const double* gt, const double* tangent,
                      const double* u, double lambda, double floor_, double* loss_out,
                      int by0 = 0, int by1 = 0, int gy0 = 0, int gy1 = 0) {
    const int P = W * H;
    SsimArgs a{};
    a.mode = mode;
    a.W = W;
    a.H = H;
    a.a = c.img.get<double>();
    a.da = tangent;
    a.b = gt;
    a.u = u;
    a.lambda = lambda;
    a.floor = floor_;
    a.adjl1 = mode == SSIM_VJP ? nullptr : img_ptr(c, c.adjl1, P);
    a.P = img_ptr(c, c.Pf, P);
    a.Q = img_ptr(c, c.Qf, P);
    a.R = img_ptr(c, c.Rf, P);
    a.by0 = by0;
    a.by1 = by1;
    if ((mode == GRAD || mode == HUTCH) && c.has_gtmom && !c.views.empty() &&
        W == c.views[0].dc.W && H == c.views[0].dc.H) {
        // a training view's target: its windowed mean / second moment are
        // fixed and were filtered once (refresh_gt_moments)
        const long long off = gt - c.gt.get<double>();
        if (off >= 0 && off % (3LL * P) == 0 && off / (3LL * P) < (long long)c.views.size())
            a.bmom = c.gtmom.get<double>() + 2 * off;
    }
    const int nb = ssim_num_blocks(W, H);
    a.loss_partials = c.partials.as<double>(std::max(nb, 10 * tr_num_blocks(c.K) + 8));
    {
        Timed t(c, KC_SSIM);
        launch_ssim(c.st, a);
        c.launches += 1;
        if (mode == GRAD && loss_out) {
            launch_sum_partials(c.st, a.loss_partials, nb, loss_out);
            c.launches += 1;
        }
    }
    Timed t(c, KC_GATHER);
    launch_ssim_gather(c.st, W, H, c.img.get<double>(), gt, a.adjl1, a.P, a.Q, a.R,
                       img_ptr(c, c.adj, P), gy0, gy1);
    c.launches += 1;
}

void check_views(Ctx& c, bool need_gt) {
    if (c.views.empty()) throw invalid("no views set");
    if (need_gt && !c.has_gt) throw invalid("views have no target images");
}

// the windowed mean and second moment of every training target (k_ssim
// BMOM), reused by every GRAD / HUTCH SSIM pass over that view
void refresh_gt_moments(Ctx& c) {
    c.has_gtmom = false;
    if (c.views.empty() || !c.has_gt) return;
    const int W = c.views[0].dc.W, H = c.views[0].dc.H;
    if (W < 6 || H < 6) return;
    const long long P = (long long)W * H;
    double* m = c.gtmom.as<double>(6 * P * c.views.size());
    for (size_t v = 0; v < c.views.size(); ++v) {
        SsimArgs a{};
        a.mode = BMOM;
        a.W = W;
        a.H = H;
        a.a = c.gt.get<double>() + 3 * P * v;
        a.b = a.a;
        a.out0 = m + 6 * P * v;
        a.out1 = m + 6 * P * v + 3 * P;
        launch_ssim(c.st, a);
        c.launches += 1;
    }
    c.has_gtmom = true;
}

const double* view_gt(Ctx& c, int v) {
    const long long P = (long long)c.views[0].dc.W * c.views[0].dc.H;
    return c.gt.get<double>() + 3 * P * v;
}

void check_ssim_size(int w, int h) {
    if (w < 6 || h < 6) throw invalid("ssim: image smaller than the window");
}

// upload an interleaved host image into a planar device buffer
double* upload_planar(Ctx& c, Buf& dst, const double* host, int P) {
    double* tmp = c.vecbuf.as<double>(3LL * P);
    SGTR_CUDA(cudaMemcpyAsync(tmp, host, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, c.st));
    double* out = img_ptr(c, dst, P);
    launch_to_planar(c.st, tmp, P, out);
    c.launches += 1;
    return out;
}

void download_interleaved(Ctx& c, const double* planar, int P, double* host) {
    double* tmp = c.vecbuf.as<double>(3LL * P);
    launch_to_interleaved(c.st, planar, P, tmp);
    c.launches += 1;
    SGTR_CUDA(cudaMemcpyAsync(host, tmp, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, c.st));
    SGTR_CUDA(cudaStreamSynchronize(c.st));
}

void ensure_tail(Ctx& c, size_t n) {
    if (c.htail_n >= n) return;
    if (c.htail) cudaFreeHost(c.htail);
    SGTR_CUDA(cudaMallocHost(&c.htail, sizeof(double) * n));
    c.htail_n = n;
}

// In-process communicator: n host threads on one GPU, one context each
// (sgtr_comm_init_loopback).  It runs the multi-rank data plane -- the view
// split, the fused [g | loss | flags | z.w] buffer, refresh bands, the sharded
// radii -- with the collectives done through device memory: every rank
// publishes its buffer, the host threads meet at a barrier, and each rank
// sums the buffers in rank order (or copies the other ranks' shards).  Tests
// use it to check the N-rank step against the 1-rank step on one GPU; the
// product path is NCCL.
struct RankPtrs {
    const double* p[8];
};
__global__ void k_sum_ranks(RankPtrs in, int n, double* __restrict__ out, long long count) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    double s = in.p[0][i];
    for (int r = 1; r < n; ++r) s += in.p[r][i];
    out[i] = s;
}

void allreduce(Ctx& c, double* buf, size_t n) {
    if (!c.collective() || n == 0) return;
    if (c.loop) {
        LoopGroup& g = *c.loop;
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        g.ptr[c.rank] = buf;
        g.barrier();
        RankPtrs rp{};
        for (int r = 0; r < g.n; ++r) rp.p[r] = g.ptr[r];
        double* tmp = c.loopbuf.as<double>(n);
        k_sum_ranks<<<(unsigned)((n + 255) / 256), 256, 0, c.st>>>(rp, g.n, tmp, (long long)n);
        SGTR_CUDA(cudaGetLastError());
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        g.barrier();  // every rank has read every buffer
        SGTR_CUDA(cudaMemcpyAsync(buf, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.st));
        c.launches += 1;
        return;
    }
    g_nccl.check(g_nccl.all_reduce(buf, buf, n, /*ncclFloat64*/ 8, /*ncclSum*/ 0, c.comm, c.st),
                 "ncclAllReduce");
}

// rank r's block [r B, (r + 1) B) of S is gathered to every rank
void allgather(Ctx& c, double* S, long long B) {
    if (c.loop) {
        LoopGroup& g = *c.loop;
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        g.ptr[c.rank] = S;
        g.barrier();
        for (int r = 0; r < g.n; ++r)
            if (r != c.rank)
                SGTR_CUDA(cudaMemcpyAsync(S + B * r, g.ptr[r] + B * r, sizeof(double) * B,
                                          cudaMemcpyDeviceToDevice, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        g.barrier();
        return;
    }
    g_nccl.check(g_nccl.all_gather(S + B * c.rank, S, B, /*ncclFloat64*/ 8, c.comm, c.st),
                 "ncclAllGather");
}

// ------------------------------------------------------------------ Algorithm 1
// One step with its draws given.  `draws` (if any) carries the Rng states to
// restore when the step fails: inside the gradient phase the reference throws
// before drawing S2 and the probes; at Hutchinson sample s it has drawn
// probes 0..s only.
// `kind` selects the update (TrArgs::kind): 0 the 3DGS2-TR Newton step,
// 1 ADAM, 2 ADAM-TR; the ADAM kinds never refresh.
void step_core(Ctx& c, const sgtr_optimizer_options& o, const std::vector<int>& s1,
               const std::vector<int>& s2, const std::vector<uint32_t>& zbits, int nu,
               bool refresh, const StepDraws* draws, sgtr_step_diagnostics* diag, int kind = 0,
               const sgtr_adam_options* adam = nullptr) {
    const int M = (int)c.views.size();
    const int W = c.views[0].dc.W, H = c.views[0].dc.H, P = W * H;
    const long long dim = c.dim();
    const long long m = 6LL * P * M;
    const RenderP ro = render_params(o.render);
    const int n1 = (int)s1.size(), n2 = refresh ? (int)s2.size() : 0;
    c.fail_sample = -1;
    // fused buffer, summed by one allreduce per step:
    //   [g_acc (dim) | loss[n1] | gflag[n1] | hflag[nu] | err_kind[n1+n2] |
    //    err_index[n1+n2] | n_dup[n1+n2] | overflows | w_acc (dim, refresh steps only)]
    // The views render without host round trips (render_view's deferred
    // mode): their errors, duplicate totals and capacity overflows arrive
    // here, read once per step.  A step in which some view (on any rank)
    // outgrew the duplicate capacity is rerun with the capacity grown to the
    // largest total -- before anything but device scratch has changed.
    const int nflag = refresh ? nu : 1;
    const size_t tail_n = 2 * n1 + nflag + 3 * (n1 + n2) + 1;
    const size_t tail_off = dim;
    double* fused = c.fused.as<double>(2 * dim + tail_n);
    double* g_acc = fused;
    double* tail = fused + tail_off;
    double* w_acc = tail + tail_n;
    double* loss = tail;
    double* gflag = tail + n1;
    double* hflag = tail + 2 * n1;
    double* errk = tail + 2 * n1 + nflag;
    double* erri = errk + (n1 + n2);
    double* ndup = erri + (n1 + n2);
    double* novf = ndup + (n1 + n2);
    const size_t fused_n = dim + tail_n + (refresh ? dim : 0);
    ensure_tail(c, tail_n);
    NvtxRange step_range("sgtr step");
    int reruns = 0;
    for (;;) {
    SGTR_CUDA(cudaMemsetAsync(fused, 0, sizeof(double) * fused_n, c.st));
    // gradient phase: stochastic_gradient (optimizer.cpp:36-65), views of S1
    // split round-robin over ranks (sgtr_shard_views).  Local view li adds
    // its gradient into accumulator li % 2 and accumulator 1 is added to
    // accumulator 0 at the end, whatever the lane count, so the summation
    // order -- and every bit of g -- does not depend on SGTR_LANES.  With two
    // lanes (streams with their own workspace) view li runs on lane li % 2,
    // so each accumulator has one writer.
    struct LaneReset {  // an exception mid-loop must not leave lane 1 current
        Ctx& c;
        ~LaneReset() { use_lane(c, 0); }
    } lane_reset{c};
    int n_local = 0;
    for (int p = c.rank; p < n1; p += c.nranks) ++n_local;
    const int lanes = std::min(n_local, lanes_knob());
    const int slots = std::min(n_local, 2);
    double* gl[2] = {g_acc, nullptr};
    if (slots > 1) {
        gl[1] = c.gacc[1].as<double>(std::max<long long>(dim, 1));
        SGTR_CUDA(cudaEventRecord(c.ev_fork, c.st));
        cudaStream_t ls = lanes > 1 ? lane_stream(c, 1) : c.st;
        if (lanes > 1) SGTR_CUDA(cudaStreamWaitEvent(ls, c.ev_fork, 0));
        SGTR_CUDA(cudaMemsetAsync(gl[1], 0, sizeof(double) * dim, ls));
    }
    int li = 0;
    for (int p = c.rank; p < n1; p += c.nranks, ++li) {
        use_lane(c, li % lanes);
        NvtxRange view_range("gradient view");
        const View& v = c.views[s1[p]];
        const ViewSlots vslots{errk + p, erri + p, ndup + p, novf};
        const ViewRender vr = render_view(c, v.dc, ro, false, 0, -1, &vslots);
        residual_adjoint(c, GRAD, W, H, view_gt(c, s1[p]), nullptr, nullptr, o.residual.lambda,
                         o.residual.floor, loss + p);
        backward_view(c, v.dc, ro, vr, 0, nullptr, nullptr, gl[li % 2], gflag + p);
    }
    if (slots > 1) {
        use_lane(c, 0);
        if (lanes > 1) {
            SGTR_CUDA(cudaEventRecord(c.ev_join[1], lane_stream(c, 1)));
            SGTR_CUDA(cudaStreamWaitEvent(c.st, c.ev_join[1], 0));
        }
        launch_add(c.st, g_acc, gl[1], dim);
        c.launches += 1;
    }
    // Hutchinson phase (optimizer.cpp:75-104), views of S2 split over ranks
    if (refresh) {
        const long long words = (dim + 31) / 32;
        uint32_t* dz = c.zbits.as<uint32_t>(std::max<long long>(words * nu, 1));
        SGTR_CUDA(cudaMemcpyAsync(dz, zbits.data(), sizeof(uint32_t) * words * nu,
                                  cudaMemcpyHostToDevice, c.st));
        // Work items: whole S2 views round-robin over ranks when there are
        // enough of them; otherwise every view is cut into B bands of tile
        // rows (B = ranks x refresh_bands) and rank r takes the bands
        // b = r (mod ranks).  A band renders its rows plus one tile row of
        // halo each side (the residual chain reaches 10 px: SSIM window 5 px
        // forward, its transpose 5 px back), evaluates SSIM on the band
        // +- 1 block row, gathers the adjoint on the band rows only and runs
        // the VJP on the band tiles, so the bands' sums add up to the view's.
        const int tiles_y = ceil_div(H, kTile);
        const bool by_view = c.refresh_bands <= 1 && n2 >= c.nranks;
        const int B = by_view ? 1 : std::min(tiles_y, c.nranks * c.refresh_bands);
        for (int s = 0; s < nu; ++s) {
            const uint32_t* zb = dz + words * s;
            for (int q = 0; q < n2; ++q) {
                if (by_view && q % c.nranks != c.rank) continue;
                for (int band = 0; band < B; ++band) {
                    if (!by_view && band % c.nranks != c.rank) continue;
                    const int tr0 = band * tiles_y / B, tr1 = (band + 1) * tiles_y / B;
                    if (tr1 <= tr0) continue;
                    const int r0 = std::max(0, tr0 - 1), r1 = std::min(tiles_y, tr1 + 1);
                    const View& v = c.views[s2[q]];
                    NvtxRange view_range("hutchinson view");
                    // the view's status is reported by its band 0 only (one
                    // writer per slot across ranks: the tail is summed)
                    ViewSlots vslots{nullptr, nullptr, nullptr, novf};
                    if (band == 0) vslots = {errk + n1 + q, erri + n1 + q, ndup + n1 + q, novf};
                    const ViewRender vr = B == 1 ? render_view(c, v.dc, ro, false, 0, -1, &vslots)
                                                 : render_view(c, v.dc, ro, false, r0, r1, &vslots);
                    double* trec = c.trec.as<double>((size_t)kTRec * (c.K + 1));
                    {
                        Timed t(c, KC_PROJECT_JVP);
                        launch_project_jvp(c.st, c.X(), c.K, c.nb, v.dc, ro, nullptr, zb, trec);
                    }
                    {
                        Timed t(c, KC_RASTER_JVP);
                        launch_raster_jvp(c.st, vr.tl, c.rec.get<double>(), trec, W, H, ro,
                                          img_ptr(c, c.tan, P));
                    }
                    c.launches += 2;
                    if (B == 1) {
                        residual_adjoint(c, HUTCH, W, H, view_gt(c, s2[q]), c.tan.get<double>(),
                                         nullptr, o.residual.lambda, o.residual.floor, nullptr);
                        backward_view(c, v.dc, ro, vr, 1, nullptr, zb, w_acc, hflag + s);
                    } else {
                        residual_adjoint(c, HUTCH, W, H, view_gt(c, s2[q]), c.tan.get<double>(),
                                         nullptr, o.residual.lambda, o.residual.floor, nullptr,
                                         r0, r1, tr0, tr1);
                        ViewRender vb = vr;
                        vb.tl.row0 = tr0;
                        vb.tl.row1 = tr1;
                        // the length order covers the whole frame; a band
                        // walks its own tile rows in row-major order
                        vb.tl.order = nullptr;
                        backward_view(c, v.dc, ro, vb, 1, nullptr, zb, w_acc, hflag + s);
                    }
                }
            }
        }
    }
    allreduce(c, fused, fused_n);
    SGTR_CUDA(cudaMemcpyAsync(c.htail, tail, sizeof(double) * tail_n, cudaMemcpyDeviceToHost,
                              c.st));
    SGTR_CUDA(cudaStreamSynchronize(c.st));
    if (c.htail[tail_n - 1] == 0.0) break;
    double need = 0.0;
    for (int j = 0; j < n1 + n2; ++j) need = std::max(need, c.htail[2 * n1 + nflag + 2 * (n1 + n2) + j]);
    if (need > (double)INT_MAX) throw Error(SGTR_RUNTIME, "binning: more than 2^31 tile duplicates");
    c.dup_cap = std::max(c.dup_cap, grow_cap((long long)need));
    ++reruns;
    }
    const double* ht = c.htail;
    const double* hk = ht + 2 * n1 + nflag;
    const double* hi = hk + (n1 + n2);
    // gradient-phase failures: nothing but t and the S1 draw has happened
    for (int p = 0; p < n1; ++p) {
        if (hk[p] != 0.0 || ht[n1 + p] != 0.0) {
            if (draws) {
                c.prefetch.reset();
                c.rng = draws->after_s1;
            }
            if (hk[p] == 1.0)
                throw numeric("rasterize: non-finite parameter in splat " +
                              std::to_string((long long)hi[p]));
            if (hk[p] == 2.0) throw invalid("quat_to_rotation: degenerate quaternion");
            throw numeric("stochastic_gradient: non-finite gradient from view " +
                          std::to_string(c.views[s1[p]].cam.id));
        }
    }
    double loss_sum = 0.0;
    for (int p = 0; p < n1; ++p) loss_sum += ht[p];
    diag->batch_loss = loss_sum * static_cast<double>(M) / (2.0 * static_cast<double>(m) * n1);
    int hutch_err = 0;
    long long hutch_idx = 0;
    bool hutch_fail = false;
    int fail_sample = 0;  // the reference throws at the first failing sample
    if (refresh) {
        for (int q = 0; q < n2 && !hutch_err; ++q)
            if (hk[n1 + q] != 0.0) {
                hutch_err = (int)hk[n1 + q];
                hutch_idx = (long long)hi[n1 + q];
            }
        hutch_fail = hutch_err != 0;  // a render error fails sample 0
        for (int s = 0; s < nu && !hutch_fail; ++s)
            if (ht[2 * n1 + s] != 0.0) {
                hutch_fail = true;
                fail_sample = s;
            }
        if (hutch_fail) c.fail_sample = fail_sample;
        if (hutch_fail && draws && fail_sample < (int)draws->after_probe.size()) {
            c.prefetch.reset();
            c.rng = draws->after_probe[fail_sample];
        }
    }
    // K14
    NvtxRange update_range("trust-region update");
    double eps = -1.0;
    if (kind != 1) {
        if (!(o.eps_start >= o.eps_end) || !(o.eps_end > 0.0))
            throw invalid("eps_at: bad schedule");
        sgtr_eps_at(o.eps_start, o.eps_end, o.total_steps, (int)c.t, &eps);
    }
    TrArgs a{};
    a.kind = kind;
    a.nb = c.nb;
    if (kind != 0) {
        // adam_direction's scalars (optimizer.cpp:159-169), host std::pow as
        // in the reference
        const long long n = std::max<long long>(dim, 1);
        a.adam_m = c.adam_m.as<double>(n);
        a.adam_v = c.adam_v.as<double>(n);
        a.beta1 = adam->beta1;
        a.beta2 = adam->beta2;
        a.adam_eps = adam->eps;
        a.bc1 = 1.0 - std::pow(adam->beta1, static_cast<double>(c.t));
        a.bc2 = 1.0 - std::pow(adam->beta2, static_cast<double>(c.t));
        const double span = std::max(1, adam->lr_position_decay_steps);
        const double frac = std::min(1.0, static_cast<double>(c.t) / span);
        a.lr[0] = adam->scene_extent * adam->lr_position *
                  std::pow(adam->lr_position_final / adam->lr_position, frac);
        a.lr[1] = adam->lr_scale;
        a.lr[2] = adam->lr_rotation;
        a.lr[3] = adam->lr_opacity;
        a.lr[4] = adam->lr_color;
    }
    a.K = c.K;
    a.x = c.X();
    a.x_out = c.x_alt.as<double>(std::max<long long>(dim, 1));
    a.g_acc = g_acc;
    a.gscale = static_cast<double>(M) / (static_cast<double>(m) * n1);
    a.g_hat = c.ghat.get<double>();
    a.d_hat = c.dhat.get<double>();
    a.w_acc = w_acc;
    a.dscale = refresh ? static_cast<double>(M) / (static_cast<double>(m) * n2 * nu) : 0.0;
    a.refresh = refresh && !hutch_fail;
    a.ghat_only = hutch_fail;
    a.theta1 = o.theta1;
    a.theta2 = o.theta2;
    a.gamma_d = o.gamma_d;
    a.eps = eps;
    const double caps[5] = {o.cap_mean, o.cap_scale, o.cap_rotation, o.cap_opacity, o.cap_color};
    const double bounds[5] = {o.s_min, o.alpha_min, o.alpha_max, o.c_min, o.c_max};
    std::copy(caps, caps + 5, a.caps);
    std::copy(bounds, bounds + 5, a.bounds);
    c.have_applied = o.record_applied_step != 0;
    a.applied = c.have_applied ? c.applied.as<double>(std::max<long long>(dim, 1)) : nullptr;
    const int nb = tr_num_blocks(c.K);
    a.partials = c.partials.as<double>(std::max(10 * nb + 8, ssim_num_blocks(W, H)));
    a.dx_buf = c.dxbuf.as<double>(std::max<long long>(dim, 1));
    a.eta_buf = c.etabuf.as<double>(std::max<long long>(dim, 1));
    a.queue = c.queue.as<int>(std::max(4LL * c.K, 1LL));
    a.queue_count = &c.dstat->queue_count;
    c.hstat->bad_index = INT_MAX;
    c.hstat->degenerate = 0;
    SGTR_CUDA(cudaMemcpyAsync(&c.dstat->bad_index, &c.hstat->bad_index, 2 * sizeof(int),
                              cudaMemcpyHostToDevice, c.st));
    a.bad_index = &c.dstat->bad_index;
    a.degenerate_flag = &c.dstat->degenerate;
    // The elementwise part (EMAs, direction, clip, apply) runs on all splats
    // on every rank; the radii -- the expensive part: Hellinger radii,
    // rotation certification and bisection -- are sharded over ranks by splat
    // range and all-gathered before the clip (multi-GPU), or computed shard
    // by shard on one rank (sgtr_set_tr_shards, which exercises the same
    // staging).  Radii are per splat, so the result does not depend on the
    // sharding.
    const bool multi = c.collective() && a.kind != 1 && !a.ghat_only;
    const int shards = multi ? c.nranks : (a.kind != 1 && !a.ghat_only ? c.tr_shards : 1);
    const long long Kp = (c.K + shards - 1) / shards;
    auto shard_range = [&](int r, int& i0, int& n) {
        const long long lo = std::min<long long>((long long)r * Kp, c.K);
        const long long hi = std::min<long long>(lo + Kp, c.K);
        i0 = (int)lo;
        n = (int)(hi - lo);
    };
    const int r_first = multi ? c.rank : 0, r_last = multi ? c.rank : shards - 1;
    for (int r = r_first; r <= r_last; ++r) {
        shard_range(r, a.i0, a.n);
        a.elementwise = r == r_first;
        {
            Timed t(c, KC_TR_UPDATE);
            launch_tr_update(c.st, a, 0);
        }
        {
            Timed t(c, KC_TR_ROT);
            launch_tr_update(c.st, a, 3);
        }
        {
            Timed t(c, KC_TR_BISECT);
            launch_tr_update(c.st, a, 1);
        }
        c.launches += 3;
    }
    if (shards > 1) {
        // Only the rotation radii live in eta_buf (K14a clips the other
        // coordinates itself), and a shard's are one contiguous block of the
        // rotation group, at the same offset in a shard-major staging buffer
        // of 4 Kp doubles per shard: copy in, all-gather over ranks (equal
        // blocks; the last shard's tail is padding), copy back.
        const long long B = 4 * Kp;
        double* S = c.stage.as<double>(std::max<long long>(B * shards, 1));
        double* rot = a.eta_buf + 6LL * c.K;
        for (int r = r_first; r <= r_last; ++r) {
            int i0, n;
            shard_range(r, i0, n);
            if (n > 0)
                SGTR_CUDA(cudaMemcpyAsync(S + B * r, rot + 4LL * i0, sizeof(double) * 4 * n,
                                          cudaMemcpyDeviceToDevice, c.st));
        }
        if (multi) allgather(c, S, B);
        if (c.K > 0)
            SGTR_CUDA(cudaMemcpyAsync(rot, S, sizeof(double) * 4 * c.K, cudaMemcpyDeviceToDevice,
                                      c.st));
    }
    {
        Timed t(c, KC_TR_APPLY);
        launch_tr_update(c.st, a, 2);
        launch_tr_finalize(c.st, a.partials, nb, c.dstat->tr);
    }
    c.launches += 2;
    SGTR_CUDA(cudaMemcpyAsync(&c.hstat->bad_index, &c.dstat->bad_index,
                              offsetof(DevStatus, scalar) - offsetof(DevStatus, bad_index),
                              cudaMemcpyDeviceToHost, c.st));
    SGTR_CUDA(cudaStreamSynchronize(c.st));
    harvest_timing(c);
    diag->gnorm = std::sqrt(c.hstat->tr[0]);
    diag->refreshed = refresh ? 1 : 0;
    diag->reruns = reruns;
    diag->n_local_views = 0;
    for (int p = c.rank; p < n1; p += c.nranks) ++diag->n_local_views;
    if (hutch_fail) {
        if (hutch_err == 1)
            throw numeric("rasterize: non-finite parameter in splat " + std::to_string(hutch_idx));
        if (hutch_err == 2) throw invalid("quat_to_rotation: degenerate quaternion");
        throw numeric("hutchinson_diag: non-finite sample");
    }
    diag->step_pre = std::sqrt(c.hstat->tr[1]);
    if (c.hstat->degenerate) throw invalid("quat_to_rotation: degenerate quaternion");
    if (c.hstat->bad_index != INT_MAX)
        throw numeric(std::string("non-finite update in group ") +
                      kGroupNames[group_of(c.K, c.hstat->bad_index)]);
    diag->step_post = std::sqrt(c.hstat->tr[2]);
    if (kind != 1) {  // apply_clipped fills the trust-region fields
        diag->eps = eps;
        diag->clip_frac = dim ? c.hstat->tr[3] / static_cast<double>(dim) : 0.0;
        diag->max_step_over_radius = c.hstat->tr[4];
    }
    std::swap(c.x.p, c.x_alt.p);
    std::swap(c.x.bytes, c.x_alt.bytes);
}

// OptimizerState(dim, seed)'s vectors (optimizer.hpp:58-72): g_hat, d_hat,
// adam_m, adam_v all zero
void zero_state(Ctx& c) {
    const long long n = std::max<long long>(c.dim(), 1);
    for (Buf* b : {&c.ghat, &c.dhat, &c.adam_m, &c.adam_v})
        SGTR_CUDA(cudaMemsetAsync(b->as<double>(n), 0, sizeof(double) * n, c.st));
}

void validate_opts(const sgtr_optimizer_options& o) {
    if (o.hutch_samples < 1) throw invalid("hutchinson_diag: nu must be >= 1");
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SGTR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("out of host memory: ") + e.what();
        return SGTR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SGTR_RUNTIME;
    }
}

Ctx& ctx_ref(sgtr_ctx* c) {
    if (!c) throw invalid("null context");
    return *reinterpret_cast<Ctx*>(c);
}

void need_scene(Ctx& c) {
    if (!c.x.p && c.K > 0) throw invalid("scene not set");
}

}  // namespace
}  // namespace sgtr

using namespace sgtr;

extern "C" {

const char* sgtr_last_error(void) { return g_last_error.c_str(); }

int sgtr_create(int device, sgtr_ctx** out) {
    return guarded([&] {
        int n = 0;
        SGTR_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw invalid("sgtr_create: no such CUDA device");
        Ctx* c = new Ctx();
        c->device = device;
        try {
            bind(*c);
            SGTR_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
            SGTR_CUDA(cudaMalloc(&c->dstat, sizeof(DevStatus)));
            SGTR_CUDA(cudaMallocHost(&c->hstat, sizeof(DevStatus)));
            for (Ctx::Lane& l : c->spare) {
                SGTR_CUDA(cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking));
                SGTR_CUDA(cudaMalloc(&l.dstat, sizeof(DevStatus)));
                SGTR_CUDA(cudaMallocHost(&l.hstat, sizeof(DevStatus)));
            }
            SGTR_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
            for (cudaEvent_t& e : c->ev_join)
                SGTR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        } catch (...) {
            delete c;
            throw;
        }
        *out = reinterpret_cast<sgtr_ctx*>(c);
    });
}

int sgtr_destroy(sgtr_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        Ctx* c = reinterpret_cast<Ctx*>(ctx);
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->st);
        delete c;
    });
}

int sgtr_get_stream(sgtr_ctx* ctx, void** stream) {
    return guarded([&] { *stream = (void*)ctx_ref(ctx).st; });
}

int sgtr_synchronize(sgtr_ctx* ctx) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int64_t sgtr_launch_count(const sgtr_ctx* ctx) {
    return ctx ? reinterpret_cast<const Ctx*>(ctx)->launches : 0;
}

namespace {
void set_scene_impl(Ctx& c, const double* x, int64_t n_splats, int sh_degree) {
    bind(c);
    if (n_splats < 0 || n_splats > (1LL << 28)) throw invalid("sgtr_set_scene: bad splat count");
    if (sh_degree < 0 || sh_degree > 3) throw invalid("sgtr_set_scene: SH degree must be 0..3");
    const int nb = (sh_degree + 1) * (sh_degree + 1) - 1;
    const bool resized = n_splats != c.K || nb != c.nb;
    c.K = (int)n_splats;
    c.nb = nb;
    const long long dim = c.dim();
    double* d = c.x.as<double>(std::max<long long>(dim, 1));
    if (dim)
        SGTR_CUDA(cudaMemcpyAsync(d, x, sizeof(double) * dim, cudaMemcpyHostToDevice, c.st));
    if (resized) zero_state(c);  // OptimizerState(dim, seed) lives with the dimension
    SGTR_CUDA(cudaStreamSynchronize(c.st));
}
}  // namespace

int sgtr_set_scene_sh(sgtr_ctx* ctx, const double* x, int64_t n_splats, int32_t sh_degree) {
    return guarded([&] { set_scene_impl(ctx_ref(ctx), x, n_splats, sh_degree); });
}

int32_t sgtr_scene_sh_degree(const sgtr_ctx* ctx) {
    if (!ctx) return -1;
    const int nb = reinterpret_cast<const Ctx*>(ctx)->nb;
    return nb == 0 ? 0 : nb == 3 ? 1 : nb == 8 ? 2 : 3;
}

int sgtr_set_scene(sgtr_ctx* ctx, const double* x, int64_t n_splats) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (n_splats < 0 || n_splats > (1LL << 28)) throw invalid("sgtr_set_scene: bad splat count");
        const long long dim = 14LL * n_splats;
        const bool resized = n_splats != c.K || c.nb != 0;
        c.K = (int)n_splats;
        c.nb = 0;
        double* d = c.x.as<double>(std::max<long long>(dim, 1));
        if (dim)
            SGTR_CUDA(cudaMemcpyAsync(d, x, sizeof(double) * dim, cudaMemcpyHostToDevice, c.st));
        if (resized) {
            // OptimizerState(dim, seed) lives with the scene dimension
            zero_state(c);
        }
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_get_scene(sgtr_ctx* ctx, double* x) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (c.dim())
            SGTR_CUDA(cudaMemcpyAsync(x, c.X(), sizeof(double) * c.dim(), cudaMemcpyDeviceToHost,
                                      c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int64_t sgtr_scene_size(const sgtr_ctx* ctx) {
    return ctx ? reinterpret_cast<const Ctx*>(ctx)->K : 0;
}

int sgtr_set_views(sgtr_ctx* ctx, const sgtr_camera* cams, int32_t n, const double* const* gts) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (n < 0) throw invalid("sgtr_set_views: negative count");
        std::vector<View> vs;
        for (int i = 0; i < n; ++i) {
            if (cams[i].width <= 0 || cams[i].height <= 0)
                throw invalid("sgtr_set_views: empty image");
            if (cams[i].width != cams[0].width || cams[i].height != cams[0].height)
                throw invalid("sgtr_set_views: all views must share one image size");
            vs.push_back({cams[i], make_devcam(cams[i])});
        }
        c.views = vs;
        c.has_gt = false;
        if (gts && n > 0) {
            const int P = cams[0].width * cams[0].height;
            double* g = c.gt.as<double>(3LL * P * n);
            for (int i = 0; i < n; ++i) {
                double* tmp = c.vecbuf.as<double>(3LL * P);
                SGTR_CUDA(cudaMemcpyAsync(tmp, gts[i], sizeof(double) * 3 * P,
                                          cudaMemcpyHostToDevice, c.st));
                launch_to_planar(c.st, tmp, P, g + 3LL * P * i);
            }
            c.has_gt = true;
        }
        refresh_gt_moments(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_render_targets(sgtr_ctx* ctx, const sgtr_render_options* ro, int32_t quantize) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        check_views(c, false);
        const int P = c.views[0].dc.W * c.views[0].dc.H;
        double* g = c.gt.as<double>(3LL * P * c.views.size());
        const RenderP rp = render_params(*ro);
        for (size_t i = 0; i < c.views.size(); ++i) {
            render_view(c, c.views[i].dc, rp, true);
            SGTR_CUDA(cudaMemcpyAsync(g + 3LL * P * i, c.img.get<double>(), sizeof(double) * 3 * P,
                                      cudaMemcpyDeviceToDevice, c.st));
            if (quantize) launch_quantize8(c.st, g + 3LL * P * i, 3LL * P);
        }
        c.has_gt = true;
        refresh_gt_moments(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_set_eval_views(sgtr_ctx* ctx, const sgtr_camera* cams, int32_t n,
                        const double* const* gts) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (n < 0) throw invalid("sgtr_set_eval_views: negative count");
        if (n > 0 && !gts) throw invalid("sgtr_set_eval_views: targets required");
        std::vector<View> vs;
        std::vector<long long> off;
        long long total = 0;
        for (int i = 0; i < n; ++i) {
            if (cams[i].width <= 0 || cams[i].height <= 0)
                throw invalid("sgtr_set_eval_views: empty image");
            vs.push_back({cams[i], make_devcam(cams[i])});
            off.push_back(total);
            total += 3LL * cams[i].width * cams[i].height;
        }
        double* g = c.eval_gt.as<double>(std::max(total, 1LL));
        for (int i = 0; i < n; ++i) {
            const int P = cams[i].width * cams[i].height;
            double* tmp = c.vecbuf.as<double>(3LL * P);
            SGTR_CUDA(cudaMemcpyAsync(tmp, gts[i], sizeof(double) * 3 * P,
                                      cudaMemcpyHostToDevice, c.st));
            launch_to_planar(c.st, tmp, P, g + off[i]);
            SGTR_CUDA(cudaStreamSynchronize(c.st));  // vecbuf is reused per view
        }
        c.eval_views = vs;
        c.eval_off = off;
    });
}

int sgtr_evaluate_scene(sgtr_ctx* ctx, int32_t which, const sgtr_render_options* ro,
                        double* view_psnr, double* view_ssim, double* mean_psnr,
                        double* mean_ssim) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        if (which != 0 && which != 1) throw invalid("evaluate_scene: bad view set");
        const std::vector<View>& vs = which == 0 ? c.eval_views : c.views;
        if (vs.empty()) throw invalid("evaluate_scene: empty view list");
        if (which == 1) check_views(c, true);
        const RenderP rp = render_params(*ro);
        const int n = (int)vs.size();
        double* sums = c.eval_sums.as<double>(2LL * n);
        for (int i = 0; i < n; ++i) {
            const int W = vs[i].dc.W, H = vs[i].dc.H, P = W * H;
            check_ssim_size(W, H);
            const double* gt = which == 0 ? c.eval_gt.get<double>() + c.eval_off[i]
                                          : view_gt(c, i);
            // quantize8(rasterize(scene, cam).color) (harness.cpp:50)
            render_view(c, vs[i].dc, rp, true);
            launch_quantize8(c.st, c.img.get<double>(), 3LL * P);
            SsimArgs a{};
            a.mode = EVAL;
            a.W = W;
            a.H = H;
            a.a = c.img.get<double>();
            a.b = gt;
            const int nb = ssim_num_blocks(W, H);
            a.loss_partials = c.partials.as<double>(2LL * nb);
            launch_ssim(c.st, a);
            launch_sum_partials(c.st, a.loss_partials, nb, sums + 2 * i);
            launch_sum_partials(c.st, a.loss_partials + nb, nb, sums + 2 * i + 1);
            c.launches += 4;
        }
        std::vector<double> h(2LL * n);
        SGTR_CUDA(cudaMemcpyAsync(h.data(), sums, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost,
                                  c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        double mp = 0.0, ms = 0.0;
        for (int i = 0; i < n; ++i) {
            const double cnt = 3.0 * vs[i].dc.W * vs[i].dc.H;
            // psnr (residuals.cpp:133-144), mean_ssim (ssim.cpp:170-175)
            const double mse = h[2 * i + 1] / cnt;
            const double p = mse < 1e-10 ? 100.0 : 10.0 * std::log10(1.0 / mse);
            const double sv = h[2 * i] / cnt;
            if (view_psnr) view_psnr[i] = p;
            if (view_ssim) view_ssim[i] = sv;
            mp += p;
            ms += sv;
        }
        if (mean_psnr) *mean_psnr = mp / n;
        if (mean_ssim) *mean_ssim = ms / n;
    });
}

// ------------------------------------------------------------------ files
namespace {
const double* bounds_or_default(const sgtr_param_bounds* b, double out[5]) {
    // ParamBounds defaults (scene.hpp:29-35)
    const double d[5] = {1e-6, 1e-4, 0.995, 1e-6, 1.5};
    if (b) {
        out[0] = b->s_min;
        out[1] = b->alpha_min;
        out[2] = b->alpha_max;
        out[3] = b->c_min;
        out[4] = b->c_max;
    } else {
        std::copy(d, d + 5, out);
    }
    return out;
}

struct PinnedHost {
    void* p = nullptr;
    explicit PinnedHost(size_t n) { SGTR_CUDA(cudaMallocHost(&p, std::max<size_t>(n, 8))); }
    ~PinnedHost() { cudaFreeHost(p); }
};
}  // namespace

int sgtr_save_scene_ply(sgtr_ctx* ctx, const char* path) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        if (c.nb)
            throw invalid("save_scene: SH coefficients have no place in the reference's PLY "
                          "(use sgtr_checkpoint_save)");
        const long long K = c.K, n = 14 * K;
        PinnedHost h(sizeof(double) * n);
        double* aos = c.vecbuf.as<double>(std::max(n, 1LL));
        launch_soa_to_aos(c.st, c.X(), K, aos);
        c.launches += K > 0;
        if (n)
            SGTR_CUDA(cudaMemcpyAsync(h.p, aos, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                      c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        ply_write(path, static_cast<const double*>(h.p), K);
    });
}

int sgtr_load_scene_ply(sgtr_ctx* ctx, const char* path, const sgtr_param_bounds* b) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        const PlyHeader hd = ply_read_header(path);
        const long long K = hd.count, n = 14 * K;
        if (K > (1LL << 28)) throw invalid("load_scene: too many splats");
        PinnedHost h(sizeof(double) * n);
        ply_read_payload(path, hd, static_cast<double*>(h.p));
        double* aos = c.vecbuf.as<double>(std::max(n, 1LL));
        double* soa = c.x_alt.as<double>(std::max(n, 1LL));
        if (n)
            SGTR_CUDA(cudaMemcpyAsync(aos, h.p, sizeof(double) * n, cudaMemcpyHostToDevice,
                                      c.st));
        launch_aos_to_soa(c.st, aos, K, soa);
        double bd[5];
        unsigned long long* first = reinterpret_cast<unsigned long long*>(
            c.partials.as<double>(1));
        launch_validate(c.st, soa, K, bounds_or_default(b, bd), first);
        c.launches += 2 * (K > 0);
        unsigned long long hf = ~0ull;
        SGTR_CUDA(cudaMemcpyAsync(&hf, first, sizeof(hf), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        throw_invalid_splat(hf);  // Scene::validate (scene.cpp:59-81)
        const bool resized = K != c.K;
        std::swap(c.x.p, c.x_alt.p);
        std::swap(c.x.bytes, c.x_alt.bytes);
        const bool sh_reset = c.nb != 0;
        c.K = (int)K;
        c.nb = 0;
        if (resized || sh_reset) zero_state(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_ply_save(const double* x, int64_t n_splats, const char* path) {
    return guarded([&] {
        if (n_splats < 0) throw invalid("save_scene: negative splat count");
        std::vector<double> aos(14 * n_splats);
        host_soa_to_aos(x, n_splats, aos.data());
        ply_write(path, aos.data(), n_splats);
    });
}

int sgtr_ply_load(const char* path, const sgtr_param_bounds* b, double* x, int64_t* n_splats) {
    return guarded([&] {
        const PlyHeader hd = ply_read_header(path);
        if (n_splats) *n_splats = hd.count;
        if (!x) return;
        std::vector<double> aos(14 * hd.count);
        ply_read_payload(path, hd, aos.data());
        std::vector<double> soa(14 * hd.count);
        host_aos_to_soa(aos.data(), hd.count, soa.data());
        double bd[5];
        host_validate(soa.data(), hd.count, bounds_or_default(b, bd));
        std::copy(soa.begin(), soa.end(), x);
    });
}

int sgtr_save_cameras(const char* path, const sgtr_camera* cams, const char* const* image_names,
                      int32_t n) {
    return guarded([&] {
        if (n < 0) throw invalid("save_cameras: negative count");
        save_cameras(path, cams, image_names, n);
    });
}

int sgtr_load_cameras(const char* path, sgtr_camera* cams, char* image_names, int32_t name_stride,
                      int32_t cap, int32_t* n) {
    return guarded([&] {
        const std::vector<CameraLine> cl = load_cameras(path);
        *n = (int32_t)cl.size();
        for (size_t i = 0; i < cl.size() && (int)i < cap; ++i) {
            if (cams) cams[i] = cl[i].cam;
            if (image_names && name_stride > 0) {
                char* dst = image_names + i * name_stride;
                std::strncpy(dst, cl[i].image_name.c_str(), name_stride - 1);
                dst[name_stride - 1] = 0;
            }
        }
    });
}

// Optimizer-state checkpoint (the reference only checkpoints
// the scene PLY, harness.cpp:157-164).  Layout: "SGTRCKP2", then four int64
// header fields K, t, the length of the Rng text and the SH basis count nb,
// the mt19937_64 state as its standard text form, the Rng's normal() spare
// (flag, value), then x | g_hat | d_hat | adam_m | adam_v (group-major).
int sgtr_checkpoint_save(sgtr_ctx* ctx, const char* path) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        c.prefetch.reset();
        const long long dim = c.dim();
        std::ostringstream rs;
        rs << c.rng.gen;
        const std::string rtxt = rs.str();
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(SGTR_RUNTIME, std::string("checkpoint: cannot open ") + path);
        const long long hdr[4] = {(long long)c.K, c.t, (long long)rtxt.size(), (long long)c.nb};
        out.write("SGTRCKP2", 8);
        out.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
        out.write(rtxt.data(), rtxt.size());
        const double spare[2] = {c.rng.have_spare ? 1.0 : 0.0, c.rng.spare};
        out.write(reinterpret_cast<const char*>(spare), sizeof(spare));
        std::vector<double> h(std::max(dim, 1LL));
        const double* vecs[5] = {c.X(), c.ghat.as<double>(std::max(dim, 1LL)),
                                 c.dhat.as<double>(std::max(dim, 1LL)),
                                 c.adam_m.as<double>(std::max(dim, 1LL)),
                                 c.adam_v.as<double>(std::max(dim, 1LL))};
        for (const double* v : vecs) {
            if (dim)
                SGTR_CUDA(cudaMemcpyAsync(h.data(), v, sizeof(double) * dim,
                                          cudaMemcpyDeviceToHost, c.st));
            SGTR_CUDA(cudaStreamSynchronize(c.st));
            out.write(reinterpret_cast<const char*>(h.data()), sizeof(double) * dim);
        }
        if (!out) throw Error(SGTR_RUNTIME, std::string("checkpoint: write failed for ") + path);
    });
}

int sgtr_checkpoint_load(sgtr_ctx* ctx, const char* path) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error(SGTR_RUNTIME, std::string("checkpoint: cannot open ") + path);
        char magic[8];
        long long hdr[4];
        in.read(magic, 8);
        in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
        if (!in || std::memcmp(magic, "SGTRCKP2", 8) != 0 || hdr[0] < 0 || hdr[0] > (1LL << 28) ||
            hdr[2] <= 0 ||
            hdr[2] > (1 << 20) || !(hdr[3] == 0 || hdr[3] == 3 || hdr[3] == 8 || hdr[3] == 15))
            throw Error(SGTR_RUNTIME, std::string("checkpoint: not a checkpoint file: ") + path);
        std::string rtxt(hdr[2], '\0');
        in.read(&rtxt[0], hdr[2]);
        double spare[2];
        in.read(reinterpret_cast<char*>(spare), sizeof(spare));
        const long long K = hdr[0], dim = (14 + 3 * hdr[3]) * K;
        std::vector<double> h(5 * std::max(dim, 1LL));
        in.read(reinterpret_cast<char*>(h.data()), sizeof(double) * 5 * dim);
        if (!in) throw Error(SGTR_RUNTIME, std::string("checkpoint: truncated file ") + path);
        Rng r;
        std::istringstream is(rtxt);
        is >> r.gen;
        if (!is) throw Error(SGTR_RUNTIME, std::string("checkpoint: bad Rng state in ") + path);
        r.have_spare = spare[0] != 0.0;
        r.spare = spare[1];
        c.prefetch.reset();
        c.K = (int)K;
        c.nb = (int)hdr[3];
        const long long n = std::max(dim, 1LL);
        Buf* dst[5] = {&c.x, &c.ghat, &c.dhat, &c.adam_m, &c.adam_v};
        for (int v = 0; v < 5; ++v)
            if (dim)
                SGTR_CUDA(cudaMemcpyAsync(dst[v]->as<double>(n), h.data() + v * dim,
                                          sizeof(double) * dim, cudaMemcpyHostToDevice, c.st));
            else
                dst[v]->as<double>(n);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        c.t = hdr[1];
        c.rng = r;
    });
}

int sgtr_scene_extent(const sgtr_camera* cams, int32_t n, double* out) {
    return guarded([&] { *out = scene_extent(cams, n); });
}

int sgtr_get_target(sgtr_ctx* ctx, int32_t view, double* gt) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        check_views(c, true);
        if (view < 0 || view >= (int)c.views.size()) throw invalid("sgtr_get_target: bad view");
        const int P = c.views[0].dc.W * c.views[0].dc.H;
        download_interleaved(c, view_gt(c, view), P, gt);
    });
}

int sgtr_state_reset(sgtr_ctx* ctx, uint64_t seed) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        zero_state(c);
        c.prefetch.reset();
        c.t = 0;
        c.rng = Rng(seed);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_state_set(sgtr_ctx* ctx, const double* g_hat, const double* d_hat, int64_t t) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        const long long n = c.dim();
        if (g_hat && n)
            SGTR_CUDA(cudaMemcpyAsync(c.ghat.as<double>(n), g_hat, sizeof(double) * n,
                                      cudaMemcpyHostToDevice, c.st));
        if (d_hat && n)
            SGTR_CUDA(cudaMemcpyAsync(c.dhat.as<double>(n), d_hat, sizeof(double) * n,
                                      cudaMemcpyHostToDevice, c.st));
        c.prefetch.reset();
        c.t = t;
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_state_get(sgtr_ctx* ctx, double* g_hat, double* d_hat, int64_t* t) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        const long long n = c.dim();
        if (g_hat && n)
            SGTR_CUDA(cudaMemcpyAsync(g_hat, c.ghat.get<double>(), sizeof(double) * n,
                                      cudaMemcpyDeviceToHost, c.st));
        if (d_hat && n)
            SGTR_CUDA(cudaMemcpyAsync(d_hat, c.dhat.get<double>(), sizeof(double) * n,
                                      cudaMemcpyDeviceToHost, c.st));
        if (t) *t = c.t;
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_rng_raw(sgtr_ctx* ctx, int64_t n, uint64_t* out) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        c.prefetch.reset();
        for (int64_t i = 0; i < n; ++i) out[i] = c.rng.gen();
    });
}

int sgtr_rng_new(uint64_t seed, sgtr_rng** out) {
    return guarded([&] { *out = reinterpret_cast<sgtr_rng*>(new std::mt19937_64(seed)); });
}

int sgtr_rng_draw(sgtr_rng* rng, int64_t n, uint64_t* out) {
    return guarded([&] {
        if (!rng) throw invalid("null rng");
        auto& g = *reinterpret_cast<std::mt19937_64*>(rng);
        for (int64_t i = 0; i < n; ++i) out[i] = g();
    });
}

int sgtr_rng_free(sgtr_rng* rng) {
    return guarded([&] { delete reinterpret_cast<std::mt19937_64*>(rng); });
}

int sgtr_step_3dgs2tr(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                      sgtr_step_diagnostics* diag) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        validate_opts(*opt);
        *diag = sgtr_step_diagnostics{0, 0, 0, 0, -1, -1, 0, 0, 0};
        if (opt->batch_size < 1) throw invalid("stochastic_gradient: empty batch");
        if (opt->hutch_batch_size < 1) throw invalid("hutchinson_diag: empty batch");
        DrawKey key;
        key.M = (int)c.views.size();
        key.dim = c.dim();
        key.b1 = opt->batch_size;
        key.b2 = opt->hutch_batch_size;
        key.nu = opt->hutch_samples;
        key.l = opt->hess_interval;
        const long long t_new = c.t + 1;
        StepDraws d;
        if (!c.prefetch.take(t_new, key, d)) {
            c.prefetch.reset();
            Rng r = c.rng;
            d = draw_step(r, t_new, key, nullptr);
        }
        c.t = t_new;
        c.rng = d.after;
        if (c.prefetch.exhausted()) c.prefetch.start(c.rng, t_new + 1, key);
        step_core(c, *opt, d.s1, d.s2, d.bits, opt->hutch_samples, d.refresh, &d, diag);
    });
}

int sgtr_step_3dgs2tr_explicit(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                               const int32_t* s1, int32_t n1, const int32_t* s2, int32_t n2,
                               const uint32_t* probe_bits, int32_t nu,
                               sgtr_step_diagnostics* diag) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        if (!opt || !diag) throw invalid("step_3dgs2tr: null options or diagnostics");
        *diag = sgtr_step_diagnostics{0, 0, 0, 0, -1, -1, 0, 0, 0};
        c.prefetch.reset();
        c.t += 1;
        const int M = (int)c.views.size();
        if (n1 < 1) throw invalid("stochastic_gradient: empty batch");
        if (!s1) throw invalid("stochastic_gradient: null batch");
        std::vector<int> v1(s1, s1 + n1), v2;
        for (int v : v1)
            if (v < 0 || v >= M) throw invalid("stochastic_gradient: view index out of range");
        const bool refresh = opt->hess_interval <= 1 || c.t % opt->hess_interval == 1;
        std::vector<uint32_t> bits;
        if (refresh) {
            if (nu < 1) throw invalid("hutchinson_diag: nu must be >= 1");
            if (n2 < 1) throw invalid("hutchinson_diag: empty batch");
            if (!s2) throw invalid("hutchinson_diag: null batch");
            if (!probe_bits) throw invalid("hutchinson_diag: null probe bits");
            v2.assign(s2, s2 + n2);
            for (int v : v2)
                if (v < 0 || v >= M) throw invalid("hutchinson_diag: view index out of range");
            const long long words = (c.dim() + 31) / 32;
            bits.assign(probe_bits, probe_bits + words * nu);
        }
        step_core(c, *opt, v1, v2, bits, nu, refresh, nullptr, diag);
    });
}

namespace {
// step_adam / step_adam_tr (optimizer.cpp:222-253): t += 1, one S1 draw
// (the ADAM kinds consume nothing else, optimizer.hpp:55-57), gradient,
// ADAM direction, plain or clipped update
void adam_step(sgtr_ctx* ctx, const sgtr_optimizer_options* opt, const sgtr_adam_options* adam,
               int kind, const int32_t* s1, int32_t n1, sgtr_step_diagnostics* diag) {
    Ctx& c = ctx_ref(ctx);
    bind(c);
    need_scene(c);
    check_views(c, true);
    if (!opt || !adam) throw invalid("step_adam: null options");
    *diag = sgtr_step_diagnostics{0, 0, 0, 0, -1, -1, 0, 0, 0};
    c.prefetch.reset();
    const int M = (int)c.views.size();
    std::vector<int> v1;
    if (s1) {
        if (n1 < 1) throw invalid("stochastic_gradient: empty batch");
        v1.assign(s1, s1 + n1);
        for (int v : v1)
            if (v < 0 || v >= M) throw invalid("stochastic_gradient: view index out of range");
        c.t += 1;
    } else {
        if (opt->batch_size < 1) throw invalid("stochastic_gradient: empty batch");
        c.t += 1;
        v1 = c.rng.sample(M, opt->batch_size);
    }
    step_core(c, *opt, v1, {}, {}, 1, false, nullptr, diag, kind, adam);
}
}  // namespace

int sgtr_step_adam(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                   const sgtr_adam_options* adam, sgtr_step_diagnostics* diag) {
    return guarded([&] { adam_step(ctx, opt, adam, 1, nullptr, 0, diag); });
}

int sgtr_step_adam_tr(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                      const sgtr_adam_options* adam, sgtr_step_diagnostics* diag) {
    return guarded([&] { adam_step(ctx, opt, adam, 2, nullptr, 0, diag); });
}

int sgtr_step_adam_explicit(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                            const sgtr_adam_options* adam, int32_t trust_region,
                            const int32_t* s1, int32_t n1, sgtr_step_diagnostics* diag) {
    return guarded([&] {
        if (!s1) throw invalid("step_adam: null S1");
        adam_step(ctx, opt, adam, trust_region ? 2 : 1, s1, n1, diag);
    });
}

int sgtr_optimizer_step(sgtr_ctx* ctx, int32_t kind, const sgtr_optimizer_options* opt,
                        const sgtr_adam_options* adam, sgtr_step_diagnostics* diag) {
    switch (kind) {
        case SGTR_KIND_3DGS2TR: return sgtr_step_3dgs2tr(ctx, opt, diag);
        case SGTR_KIND_ADAM: return sgtr_step_adam(ctx, opt, adam, diag);
        case SGTR_KIND_ADAM_TR: return sgtr_step_adam_tr(ctx, opt, adam, diag);
        default:
            g_last_error = "optimizer_step: unknown optimizer kind";
            return SGTR_INVALID_ARGUMENT;
    }
}

int sgtr_state_set_adam(sgtr_ctx* ctx, const double* m, const double* v) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        const long long n = c.dim();
        if (m && n)
            SGTR_CUDA(cudaMemcpyAsync(c.adam_m.as<double>(n), m, sizeof(double) * n,
                                      cudaMemcpyHostToDevice, c.st));
        if (v && n)
            SGTR_CUDA(cudaMemcpyAsync(c.adam_v.as<double>(n), v, sizeof(double) * n,
                                      cudaMemcpyHostToDevice, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_state_get_adam(sgtr_ctx* ctx, double* m, double* v) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        const long long n = c.dim();
        if (m && n)
            SGTR_CUDA(cudaMemcpyAsync(m, c.adam_m.as<double>(n), sizeof(double) * n,
                                      cudaMemcpyDeviceToHost, c.st));
        if (v && n)
            SGTR_CUDA(cudaMemcpyAsync(v, c.adam_v.as<double>(n), sizeof(double) * n,
                                      cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_step_failed_sample(sgtr_ctx* ctx, int32_t* sample) {
    return guarded([&] {
        if (!ctx || !sample) throw invalid("sgtr_step_failed_sample: null argument");
        *sample = ctx_ref(ctx).fail_sample;
    });
}

int sgtr_get_applied_step(sgtr_ctx* ctx, double* out) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (!c.have_applied) throw invalid("no applied step recorded");
        SGTR_CUDA(cudaMemcpyAsync(out, c.applied.get<double>(), sizeof(double) * c.dim(),
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

// ------------------------------------------------------------------ seams
int sgtr_rasterize(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                   double* color, double* t_final) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        render_view(c, dc, render_params(*ro), true);
        const int P = dc.W * dc.H;
        if (t_final)
            SGTR_CUDA(cudaMemcpyAsync(t_final, c.tfin.get<double>(), sizeof(double) * P,
                                      cudaMemcpyDeviceToHost, c.st));
        download_interleaved(c, c.img.get<double>(), P, color);
    });
}

int sgtr_rasterize_jvp(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                       const double* v, double* tangent) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        const RenderP rp = render_params(*ro);
        const ViewRender vr = render_view(c, dc, rp, true);
        const int P = dc.W * dc.H;
        double* dv = c.seam0.as<double>(std::max<long long>(c.dim(), 1));
        SGTR_CUDA(cudaMemcpyAsync(dv, v, sizeof(double) * c.dim(), cudaMemcpyHostToDevice, c.st));
        double* trec = c.trec.as<double>((size_t)kTRec * (c.K + 1));
        launch_project_jvp(c.st, c.X(), c.K, c.nb, dc, rp, dv, nullptr, trec);
        launch_raster_jvp(c.st, vr.tl, c.rec.get<double>(), trec, dc.W, dc.H, rp,
                          img_ptr(c, c.tan, P));
        c.launches += 2;
        download_interleaved(c, c.tan.get<double>(), P, tangent);
    });
}

int sgtr_rasterize_vjp(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                       const double* adjoint, double* grad) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        const RenderP rp = render_params(*ro);
        const ViewRender vr = render_view(c, dc, rp, true);
        const int P = dc.W * dc.H;
        upload_planar(c, c.adj, adjoint, P);
        double* g = c.seam1.as<double>(std::max<long long>(c.dim(), 1));
        SGTR_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * std::max<long long>(c.dim(), 1), c.st));
        double* flag = c.seam2.as<double>(1);
        backward_view(c, dc, rp, vr, 0, nullptr, nullptr, g, flag);
        SGTR_CUDA(cudaMemcpyAsync(grad, g, sizeof(double) * c.dim(), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

namespace {

// shared body of the SSIM / residual seams on host images
void ssim_seam(Ctx& c, int mode, const double* a, const double* da, const double* b,
               const double* u, int w, int h, double lambda, double floor_, double* out0,
               double* out1, double* adj_out) {
    bind(c);
    check_ssim_size(w, h);
    const int P = w * h;
    double* A = upload_planar(c, c.img, a, P);
    double* B = upload_planar(c, c.seam0, b, P);
    double* DA = da ? upload_planar(c, c.tan, da, P) : nullptr;
    double* U = nullptr;
    if (u && mode == RES_VJP) {
        U = c.seam1.as<double>(6LL * P);
        SGTR_CUDA(cudaMemcpyAsync(U, u, sizeof(double) * 6 * P, cudaMemcpyHostToDevice, c.st));
    } else if (u) {
        U = upload_planar(c, c.seam1, u, P);
    }
    if (mode == RES_VJP || mode == SSIM_VJP) {
        residual_adjoint(c, mode, w, h, B, DA, U, lambda, floor_, nullptr);
        download_interleaved(c, c.adj.get<double>(), P, adj_out);
        return;
    }
    SsimArgs s{};
    s.mode = mode;
    s.W = w;
    s.H = h;
    s.a = A;
    s.da = DA;
    s.b = B;
    s.lambda = lambda;
    s.floor = floor_;
    const bool resid = mode == RES_VEC || mode == RES_JVP;
    double* o0 = c.seam2.as<double>((resid ? 6LL : 6LL) * P);
    double* o1 = o0 + 3LL * P;
    s.out0 = o0;
    s.out1 = o1;
    launch_ssim(c.st, s);
    c.launches += 1;
    if (resid) {
        SGTR_CUDA(cudaMemcpyAsync(out0, o0, sizeof(double) * 6 * P, cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        return;
    }
    download_interleaved(c, o0, P, out0);
    if (out1) download_interleaved(c, o1, P, out1);
}

}  // namespace

int sgtr_ssim_map(sgtr_ctx* ctx, const double* a, const double* b, int32_t w, int32_t h,
                  double* out) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), SSIM_MAP, a, nullptr, b, nullptr, w, h, 0.0, 0.0, out, nullptr,
                  nullptr);
    });
}

int sgtr_ssim_jvp(sgtr_ctx* ctx, const double* a, const double* da, const double* b, int32_t w,
                  int32_t h, double* s, double* ds) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), SSIM_JVP, a, da, b, nullptr, w, h, 0.0, 0.0, s, ds, nullptr);
    });
}

int sgtr_ssim_vjp(sgtr_ctx* ctx, const double* a, const double* b, const double* upstream,
                  int32_t w, int32_t h, double* grad) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), SSIM_VJP, a, nullptr, b, upstream, w, h, 0.0, 0.0, nullptr,
                  nullptr, grad);
    });
}

int sgtr_residual_vector(sgtr_ctx* ctx, const double* rendered, const double* gt, int32_t w,
                         int32_t h, const sgtr_residual_options* o, double* r) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), RES_VEC, rendered, nullptr, gt, nullptr, w, h, o->lambda,
                  o->floor, r, nullptr, nullptr);
    });
}

int sgtr_residual_jvp(sgtr_ctx* ctx, const double* rendered, const double* tangent,
                      const double* gt, int32_t w, int32_t h, const sgtr_residual_options* o,
                      double* dr) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), RES_JVP, rendered, tangent, gt, nullptr, w, h, o->lambda,
                  o->floor, dr, nullptr, nullptr);
    });
}

int sgtr_residual_vjp(sgtr_ctx* ctx, const double* rendered, const double* gt, int32_t w,
                      int32_t h, const double* u, const sgtr_residual_options* o, double* adj) {
    return guarded([&] {
        ssim_seam(ctx_ref(ctx), RES_VJP, rendered, nullptr, gt, u, w, h, o->lambda, o->floor,
                  nullptr, nullptr, adj);
    });
}

int sgtr_view_jacobian_apply(sgtr_ctx* ctx, int32_t view, const double* v,
                             const sgtr_residual_options* rs, const sgtr_render_options* ro,
                             double* out) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        if (view < 0 || view >= (int)c.views.size()) throw invalid("view index out of range");
        const View& vw = c.views[view];
        const RenderP rp = render_params(*ro);
        const ViewRender vr = render_view(c, vw.dc, rp, true);
        const int W = vw.dc.W, H = vw.dc.H, P = W * H;
        check_ssim_size(W, H);
        double* dv = c.seam0.as<double>(std::max<long long>(c.dim(), 1));
        SGTR_CUDA(cudaMemcpyAsync(dv, v, sizeof(double) * c.dim(), cudaMemcpyHostToDevice, c.st));
        double* trec = c.trec.as<double>((size_t)kTRec * (c.K + 1));
        launch_project_jvp(c.st, c.X(), c.K, c.nb, vw.dc, rp, dv, nullptr, trec);
        launch_raster_jvp(c.st, vr.tl, c.rec.get<double>(), trec, W, H, rp, img_ptr(c, c.tan, P));
        SsimArgs s{};
        s.mode = RES_JVP;
        s.W = W;
        s.H = H;
        s.a = c.img.get<double>();
        s.da = c.tan.get<double>();
        s.b = view_gt(c, view);
        s.lambda = rs->lambda;
        s.floor = rs->floor;
        s.out0 = c.seam2.as<double>(6LL * P);
        launch_ssim(c.st, s);
        c.launches += 3;
        SGTR_CUDA(cudaMemcpyAsync(out, s.out0, sizeof(double) * 6 * P, cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_view_jacobian_applyT(sgtr_ctx* ctx, int32_t view, const double* u,
                              const sgtr_residual_options* rs, const sgtr_render_options* ro,
                              double* grad) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        if (view < 0 || view >= (int)c.views.size()) throw invalid("view index out of range");
        const View& vw = c.views[view];
        const RenderP rp = render_params(*ro);
        const ViewRender vr = render_view(c, vw.dc, rp, true);
        const int W = vw.dc.W, H = vw.dc.H, P = W * H;
        check_ssim_size(W, H);
        double* U = c.seam1.as<double>(6LL * P);
        SGTR_CUDA(cudaMemcpyAsync(U, u, sizeof(double) * 6 * P, cudaMemcpyHostToDevice, c.st));
        residual_adjoint(c, RES_VJP, W, H, view_gt(c, view), nullptr, U, rs->lambda, rs->floor,
                         nullptr);
        double* g = c.seam0.as<double>(std::max<long long>(c.dim(), 1));
        SGTR_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * std::max<long long>(c.dim(), 1), c.st));
        double* flag = c.seam2.as<double>(1);
        backward_view(c, vw.dc, rp, vr, 0, nullptr, nullptr, g, flag);
        SGTR_CUDA(cudaMemcpyAsync(grad, g, sizeof(double) * c.dim(), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_stochastic_gradient(sgtr_ctx* ctx, const int32_t* batch, int32_t n,
                             const sgtr_residual_options* rs, const sgtr_render_options* ro,
                             double* g, double* batch_loss) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        if (n < 1) throw invalid("stochastic_gradient: empty batch");
        const int M = (int)c.views.size();
        const int W = c.views[0].dc.W, H = c.views[0].dc.H;
        check_ssim_size(W, H);
        const long long m = 6LL * W * H * M, dim = std::max<long long>(c.dim(), 1);
        double* acc = c.seam0.as<double>(dim + 2LL * n);
        double* loss = acc + dim;
        double* flags = loss + n;
        SGTR_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * (dim + 2LL * n), c.st));
        const RenderP rp = render_params(*ro);
        for (int p = 0; p < n; ++p) {
            if (batch[p] < 0 || batch[p] >= M)
                throw invalid("stochastic_gradient: view index out of range");
            const View& v = c.views[batch[p]];
            const ViewRender vr = render_view(c, v.dc, rp, true);
            residual_adjoint(c, GRAD, W, H, view_gt(c, batch[p]), nullptr, nullptr, rs->lambda,
                             rs->floor, loss + p);
            backward_view(c, v.dc, rp, vr, 0, nullptr, nullptr, acc, flags + p);
        }
        std::vector<double> tail(2 * n);
        SGTR_CUDA(cudaMemcpyAsync(tail.data(), loss, sizeof(double) * 2 * n,
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        for (int p = 0; p < n; ++p)
            if (tail[n + p] != 0.0)
                throw numeric("stochastic_gradient: non-finite gradient from view " +
                              std::to_string(c.views[batch[p]].cam.id));
        const double scale = static_cast<double>(M) / (static_cast<double>(m) * n);
        launch_scale(c.st, acc, c.dim(), scale);
        c.launches += 1;
        SGTR_CUDA(cudaMemcpyAsync(g, acc, sizeof(double) * c.dim(), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        double loss_sum = 0.0;
        for (int p = 0; p < n; ++p) loss_sum += tail[p];
        if (batch_loss)
            *batch_loss = loss_sum * static_cast<double>(M) / (2.0 * static_cast<double>(m) * n);
    });
}

int sgtr_hutchinson_diag(sgtr_ctx* ctx, const int32_t* batch, int32_t n, int32_t nu,
                         const double* probes, const sgtr_residual_options* rs,
                         const sgtr_render_options* ro, double* d) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        check_views(c, true);
        if (nu < 1) throw invalid("hutchinson_diag: nu must be >= 1");
        if (n < 1) throw invalid("hutchinson_diag: empty batch");
        const int M = (int)c.views.size();
        const int W = c.views[0].dc.W, H = c.views[0].dc.H, P = W * H;
        check_ssim_size(W, H);
        const long long m = 6LL * P * M, dim = std::max<long long>(c.dim(), 1);
        double* acc = c.seam1.as<double>(dim + 1);
        double* flag = acc + dim;
        SGTR_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * (dim + 1), c.st));
        double* z = c.seam0.as<double>(dim);
        const RenderP rp = render_params(*ro);
        for (int s = 0; s < nu; ++s) {
            SGTR_CUDA(cudaMemcpyAsync(z, probes + s * c.dim(), sizeof(double) * c.dim(),
                                      cudaMemcpyHostToDevice, c.st));
            for (int q = 0; q < n; ++q) {
                if (batch[q] < 0 || batch[q] >= M)
                    throw invalid("hutchinson_diag: view index out of range");
                const View& v = c.views[batch[q]];
                const ViewRender vr = render_view(c, v.dc, rp, true);
                double* trec = c.trec.as<double>((size_t)kTRec * (c.K + 1));
                launch_project_jvp(c.st, c.X(), c.K, c.nb, v.dc, rp, z, nullptr, trec);
                launch_raster_jvp(c.st, vr.tl, c.rec.get<double>(), trec, W, H, rp,
                                  img_ptr(c, c.tan, P));
                c.launches += 2;
                residual_adjoint(c, HUTCH, W, H, view_gt(c, batch[q]), c.tan.get<double>(),
                                 nullptr, rs->lambda, rs->floor, nullptr);
                backward_view(c, v.dc, rp, vr, 1, z, nullptr, acc, flag);
            }
            double hf = 0.0;
            SGTR_CUDA(cudaMemcpyAsync(&hf, flag, sizeof(double), cudaMemcpyDeviceToHost, c.st));
            SGTR_CUDA(cudaStreamSynchronize(c.st));
            if (hf != 0.0) throw numeric("hutchinson_diag: non-finite sample");
        }
        const double scale = static_cast<double>(M) / (static_cast<double>(m) * n * nu);
        launch_scale(c.st, acc, c.dim(), scale);
        c.launches += 1;
        SGTR_CUDA(cudaMemcpyAsync(d, acc, sizeof(double) * c.dim(), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_shd_radii(sgtr_ctx* ctx, double eps, const double caps[5], double* eta) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        double* e = c.seam0.as<double>(std::max<long long>(c.dim(), 1));
        launch_shd_radii(c.st, c.K, c.nb, c.X(), eps, caps, e);
        c.launches += 1;
        SGTR_CUDA(cudaMemcpyAsync(eta, e, sizeof(double) * c.dim(), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_eps_at(double e0, double e1, int32_t total, int32_t t, double* out) {
    return guarded([&] {  // trust_region.cpp:261-268
        if (!(e0 >= e1) || !(e1 > 0.0)) throw invalid("eps_at: bad schedule");
        if (total <= 0 || t <= 0) {
            *out = e0;
        } else if (t >= total) {
            *out = e1;
        } else {
            const double frac = static_cast<double>(t) / total;
            *out = e0 * std::pow(e1 / e0, frac);
        }
    });
}

int sgtr_project(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                 double* out) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        double* o = c.seam0.as<double>(std::max(12LL * c.K, 1LL));
        launch_project_dump(c.st, c.X(), c.K, dc, render_params(*ro), o);
        c.launches += 1;
        SGTR_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * 12 * c.K, cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sgtr_dump_binning(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                      int32_t* n_visible, int32_t* order, int64_t* n_dup, int64_t* tile_start,
                      int64_t* tile_end, int32_t* lists) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        const ViewRender vr = render_view(c, dc, render_params(*ro), true);
        *n_visible = vr.n_visible;
        *n_dup = vr.n_dup;
        if (!lists) return;
        const int n_tiles = vr.tl.tiles_x * vr.tl.tiles_y;
        std::vector<int> ids(vr.n_visible), ts(n_tiles), te(n_tiles), dv(vr.n_dup), did(vr.n_dup);
        SGTR_CUDA(cudaMemcpyAsync(ids.data(), c.ids_alt.get<int>(), sizeof(int) * vr.n_visible,
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaMemcpyAsync(ts.data(), vr.tl.tile_start, sizeof(int) * n_tiles,
                                  cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaMemcpyAsync(te.data(), vr.tl.tile_end, sizeof(int) * n_tiles,
                                  cudaMemcpyDeviceToHost, c.st));
        if (vr.n_dup) {
            SGTR_CUDA(cudaMemcpyAsync(dv.data(), vr.tl.sorted_d, sizeof(int) * vr.n_dup,
                                      cudaMemcpyDeviceToHost, c.st));
            SGTR_CUDA(cudaMemcpyAsync(did.data(), vr.tl.dup_id, sizeof(int) * vr.n_dup,
                                      cudaMemcpyDeviceToHost, c.st));
        }
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        for (int i = 0; i < vr.n_visible; ++i) order[i] = ids[i];
        for (int t = 0; t < n_tiles; ++t) {  // empty tiles as [0, 0) (the oracle's convention)
            tile_start[t] = ts[t] == te[t] ? 0 : ts[t];
            tile_end[t] = ts[t] == te[t] ? 0 : te[t];
        }
        for (long long j = 0; j < vr.n_dup; ++j) lists[j] = did[dv[j]];
    });
}

// dataset.cpp:25-67 with the declared extensions (W != H, size scaling)
int sgtr_make_synthetic(const sgtr_synth_config* cfg, double* gt_x, double* init_x,
                        sgtr_camera* cams) {
    return guarded([&] {
        if (cfg->gt_splats < 1 || cfg->init_splats < 0 || cfg->views < 0 || cfg->width < 1 ||
            cfg->height < 1)
            throw invalid("sgtr_make_synthetic: bad configuration");
        Rng rng(cfg->seed);
        const long long kg = cfg->gt_splats, ki = cfg->init_splats;
        const double ss = cfg->size_scale;
        auto put = [](double* x, long long k, long long i, const double* mu, const double* s,
                      const double* q, double a, const double* c) {
            for (int j = 0; j < 3; ++j) {
                x[3 * i + j] = mu[j];
                x[3 * k + 3 * i + j] = s[j];
                x[11 * k + 3 * i + j] = c[j];
            }
            for (int j = 0; j < 4; ++j) x[6 * k + 4 * i + j] = q[j];
            x[10 * k + i] = a;
        };
        std::vector<double> gmu(3 * kg);
        for (long long i = 0; i < kg; ++i) {
            double mu[3], s[3], q[4], c[3];
            for (int a = 0; a < 3; ++a) mu[a] = rng.uniform(-0.5, 0.5);
            for (int a = 0; a < 3; ++a) s[a] = rng.log_uniform(0.02 * ss, 0.2 * ss);
            for (int a = 0; a < 4; ++a) q[a] = rng.normal();
            // random_unit_quat's q.norm(): Eigen's SSE2 order for a 4-vector
            const double n = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
            if (n > 1e-9) {
                for (int a = 0; a < 4; ++a) q[a] = q[a] / n;
            } else {
                q[0] = q[1] = q[2] = 0.0;
                q[3] = 1.0;
            }
            const double alpha = rng.uniform(0.3, 0.9);
            for (int a = 0; a < 3; ++a) c[a] = rng.uniform(0.1, 1.0);
            put(gt_x, kg, i, mu, s, q, alpha, c);
            for (int a = 0; a < 3; ++a) gmu[3 * i + a] = mu[a];
        }
        for (long long i = 0; i < ki; ++i) {
            double mu[3];
            const double* src = gmu.data() + 3 * (i % kg);
            for (int a = 0; a < 3; ++a) mu[a] = src[a] + cfg->sigma_init * ss * rng.normal();
            const double s[3] = {cfg->init_scale * ss, cfg->init_scale * ss, cfg->init_scale * ss};
            const double q[4] = {0, 0, 0, 1};
            const double c[3] = {0.5, 0.5, 0.5};
            put(init_x, ki, i, mu, s, q, cfg->init_opacity, c);
        }
        if (cfg->sh_degree < 0 || cfg->sh_degree > 3)
            throw invalid("sgtr_make_synthetic: SH degree must be 0..3");
        const long long nsh = 3LL * ((cfg->sh_degree + 1) * (cfg->sh_degree + 1) - 1);
        if (nsh) {
            // SH extension: GT coefficients 0.1 N(0,1) from their own stream
            // (so degree 0 data are unchanged), init coefficients 0
            Rng rs(cfg->seed + 0x5348ULL);
            for (long long t = 0; t < nsh * kg; ++t) gt_x[14 * kg + t] = 0.1 * rs.normal();
            for (long long t = 0; t < nsh * ki; ++t) init_x[14 * ki + t] = 0.0;
        }
        const double focal = cfg->focal_factor * cfg->height;
        for (int v = 0; v < cfg->views; ++v) {
            const double ang = 2.0 * M_PI * v / cfg->views;
            const double eye[3] = {cfg->camera_radius * std::cos(ang),
                                   cfg->camera_radius * std::sin(ang), cfg->camera_height};
            // look_at_camera (scene.cpp:130-147)
            double z[3] = {0.0 - eye[0], 0.0 - eye[1], 0.0 - eye[2]};  // target - eye: +0, not -0
            auto normalize = [](double* u) {
                const double n2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
                if (n2 > 0.0) {
                    const double s = std::sqrt(n2);
                    for (int i = 0; i < 3; ++i) u[i] = u[i] / s;
                }
            };
            auto cross = [](const double* a, const double* b, double* o) {
                o[0] = a[1] * b[2] - a[2] * b[1];
                o[1] = a[2] * b[0] - a[0] * b[2];
                o[2] = a[0] * b[1] - a[1] * b[0];
            };
            normalize(z);
            double up[3] = {0, 0, 1};
            if (std::abs(z[0] * up[0] + z[1] * up[1] + z[2] * up[2]) > 0.999) {
                up[1] = 1;
                up[2] = 0;
            }
            double xa[3], ya[3];
            cross(z, up, xa);
            normalize(xa);
            cross(z, xa, ya);
            const double r[9] = {xa[0], xa[1], xa[2], ya[0], ya[1], ya[2], z[0], z[1], z[2]};
            sgtr_camera cam{};
            cam.id = v;
            cam.width = cfg->width;
            cam.height = cfg->height;
            cam.fx = focal;
            cam.fy = focal;
            cam.cx = cfg->width / 2.0;
            cam.cy = cfg->height / 2.0;
            // rotation_to_quat (scene.cpp:94-128)
            double* q = cam.q_wc;
            const double tr = r[0] + (r[4] + r[8]);  // trace(): halves
            if (tr > 0.0) {
                const double s = std::sqrt(tr + 1.0) * 2.0;
                q[3] = 0.25 * s;
                q[0] = (r[7] - r[5]) / s;
                q[1] = (r[2] - r[6]) / s;
                q[2] = (r[3] - r[1]) / s;
            } else if (r[0] > r[4] && r[0] > r[8]) {
                const double s = std::sqrt(1.0 + r[0] - r[4] - r[8]) * 2.0;
                q[3] = (r[7] - r[5]) / s;
                q[0] = 0.25 * s;
                q[1] = (r[1] + r[3]) / s;
                q[2] = (r[2] + r[6]) / s;
            } else if (r[4] > r[8]) {
                const double s = std::sqrt(1.0 + r[4] - r[0] - r[8]) * 2.0;
                q[3] = (r[2] - r[6]) / s;
                q[0] = (r[1] + r[3]) / s;
                q[1] = 0.25 * s;
                q[2] = (r[5] + r[7]) / s;
            } else {
                const double s = std::sqrt(1.0 + r[8] - r[0] - r[4]) * 2.0;
                q[3] = (r[3] - r[1]) / s;
                q[0] = (r[2] + r[6]) / s;
                q[1] = (r[5] + r[7]) / s;
                q[2] = 0.25 * s;
            }
            const double qn = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
            for (int i = 0; i < 4; ++i) q[i] = q[i] / qn;
            for (int i = 0; i < 3; ++i)
                cam.t_wc[i] =  // -r * eye: a column-major product row, summed in halves
                    -r[3 * i] * eye[0] + (-r[3 * i + 1] * eye[1] + -r[3 * i + 2] * eye[2]);
            cams[v] = cam;
        }
    });
}

int sgtr_kernel_timing(sgtr_ctx* ctx, int32_t enable) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        harvest_timing(c);
        c.timer.on = enable != 0;
        for (int k = 0; k < KC_COUNT; ++k) {
            c.timer.total_ms[k] = 0.0;
            c.timer.count[k] = 0;
        }
    });
}

int sgtr_kernel_timing_report(sgtr_ctx* ctx, char* buf, int32_t len) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        harvest_timing(c);
        std::string s = "{";
        for (int k = 0; k < KC_COUNT; ++k) {
            char item[128];
            std::snprintf(item, sizeof(item), "%s\"%s\": [%lld, %.6f]", k ? ", " : "",
                          kClassNames[k], c.timer.count[k], c.timer.total_ms[k]);
            s += item;
        }
        s += "}";
        if ((int)s.size() >= len) throw invalid("sgtr_kernel_timing_report: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int sgtr_blend_stats(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                     int64_t* evaluated, int64_t* contributing) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const DevCam dc = make_devcam(*cam);
        RenderP rp = render_params(*ro);
        rp.cull = 0;  // count the reference's pairs: no contribution culling
        const ViewRender vr = render_view(c, dc, rp, true);
        unsigned long long* cnt = c.seam2.as<unsigned long long>(2);
        SGTR_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), c.st));
        const int P = dc.W * dc.H;
        launch_raster_fwd(c.st, vr.tl, c.rec.get<double>(), dc.W, dc.H, rp, img_ptr(c, c.img, P),
                          c.tfin.as<double>(P), c.last.as<int>(P), cnt);
        unsigned long long h[2];
        SGTR_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c.st));
        SGTR_CUDA(cudaStreamSynchronize(c.st));
        *evaluated = (int64_t)h[0];
        *contributing = (int64_t)h[1];
    });
}

int sgtr_view_stats(sgtr_ctx* ctx, const sgtr_camera* cam, const sgtr_render_options* ro,
                    int32_t* n_visible, int64_t* n_dup) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        need_scene(c);
        const ViewRender vr = render_view(c, make_devcam(*cam), render_params(*ro), true);
        *n_visible = vr.n_visible;
        *n_dup = vr.n_dup;
    });
}

int sgtr_fp64_peak(int device, double* tflops) {
    return guarded([&] { *tflops = fp64_fma_peak_tflops(device); });
}

int sgtr_check_fast_exp(int64_t n, double lo, double hi, uint64_t seed, int64_t* mismatches) {
    return guarded([&] {
        if (n < 0 || !(lo <= hi)) throw invalid("check_fast_exp: bad range");
        *mismatches = fast_exp_mismatches(n, lo, hi, seed);
    });
}

int sgtr_shard_views(int32_t n, int32_t rank, int32_t nranks, int32_t* positions,
                     int32_t* count) {
    return guarded([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw invalid("sgtr_shard_views: bad rank");
        int m = 0;
        for (int p = rank; p < n; p += nranks) {  // the loop step_core runs
            if (positions) positions[m] = p;
            ++m;
        }
        *count = m;
    });
}

int sgtr_nccl_unique_id(uint8_t out[128]) {
    return guarded([&] {
        g_nccl.load();
        g_nccl.check(g_nccl.get_unique_id(out), "ncclGetUniqueId");
    });
}

int sgtr_set_dup_capacity(sgtr_ctx* ctx, int64_t capacity) {
    return guarded([&] {
        if (capacity < 0) throw invalid("sgtr_set_dup_capacity: negative capacity");
        if (capacity > INT_MAX) throw invalid("sgtr_set_dup_capacity: more than 2^31 entries");
        ctx_ref(ctx).dup_cap = capacity;
    });
}

int sgtr_set_refresh_bands(sgtr_ctx* ctx, int32_t bands_per_rank) {
    return guarded([&] {
        if (bands_per_rank < 1) throw invalid("sgtr_set_refresh_bands: need >= 1 band");
        ctx_ref(ctx).refresh_bands = bands_per_rank;
    });
}

int sgtr_set_tr_shards(sgtr_ctx* ctx, int32_t shards) {
    return guarded([&] {
        if (shards < 1) throw invalid("sgtr_set_tr_shards: need >= 1 shard");
        ctx_ref(ctx).tr_shards = shards;
    });
}

int sgtr_loopback_group_create(int32_t nranks, sgtr_group** out) {
    return guarded([&] {
        if (!out) throw invalid("sgtr_loopback_group_create: null output");
        if (nranks < 1 || nranks > 8) throw invalid("sgtr_loopback_group_create: 1..8 ranks");
        *out = reinterpret_cast<sgtr_group*>(new LoopGroup(nranks));
    });
}

int sgtr_loopback_group_destroy(sgtr_group* g) {
    return guarded([&] { delete reinterpret_cast<LoopGroup*>(g); });
}

int sgtr_comm_init_loopback(sgtr_ctx* ctx, sgtr_group* group, int32_t rank) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (!group) throw invalid("sgtr_comm_init_loopback: null group");
        LoopGroup* g = reinterpret_cast<LoopGroup*>(group);
        if (rank < 0 || rank >= g->n) throw invalid("sgtr_comm_init: bad rank");
        if (c.comm || c.loop) throw invalid("sgtr_comm_init: communicator already initialised");
        c.loop = g;
        c.nranks = g->n;
        c.rank = rank;
    });
}

int sgtr_comm_init(sgtr_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank) {
    return guarded([&] {
        Ctx& c = ctx_ref(ctx);
        bind(c);
        if (nranks < 1 || rank < 0 || rank >= nranks) throw invalid("sgtr_comm_init: bad rank");
        if (!id) throw invalid("sgtr_comm_init: null unique id");
        if (c.comm || c.loop) throw invalid("sgtr_comm_init: communicator already initialised");
        // a 1-rank communicator is created too (it runs the same allreduce
        // path; tests use it to exercise the NCCL plumbing on one GPU)
        g_nccl.load();
        auto init = (CommInitRankFn)dlsym(g_nccl.lib, "ncclCommInitRank");
        if (!init) throw Error(SGTR_RUNTIME, "libnccl.so.2 lacks ncclCommInitRank");
        UniqueId u;
        std::memcpy(u.internal, id, 128);
        void* comm = nullptr;
        g_nccl.check(init(&comm, nranks, u, rank), "ncclCommInitRank");
        // the view split only changes once the communicator exists: a failed
        // init leaves the context a single-rank one
        c.comm = comm;
        c.nranks = nranks;
        c.rank = rank;
    });
}

}  // extern "C"
