// vcs_device.cuh — device-side internals shared by the builder, solver and greedy units.
#pragma once

#include "vcs_internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#define VCS_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t err_ = (call);                                                             \
        if (err_ != cudaSuccess)                                                               \
            ::vcs::raise(VCS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(err_));     \
    } while (0)

#define VCS_LAUNCHED()                                                                         \
    do {                                                                                       \
        cudaError_t err_ = cudaGetLastError();                                                 \
        if (err_ != cudaSuccess)                                                               \
            ::vcs::raise(VCS_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(err_)); \
        ::vcs::note_launch();                                                                  \
        ::vcs::debug_sync_check(__FILE__, __LINE__);                                           \
    } while (0)

namespace vcs {

constexpr uint32_t kEmpty32 = 0xffffffffu;

// VCS_SYNC_CHECK (debugging): synchronise after every launch that is not being captured and
// report the launch site of an asynchronous fault.
void debug_sync_check(const char* file, int line);
extern thread_local bool g_capturing; // set while a solve graph is being captured

// Configure the device's default memory pool once so freed blocks stay cached for reuse
// (building and freeing spaces repeatedly then costs no cudaMalloc / implicit device sync).
void init_pool(int device);

// Device allocation on the stream-ordered pool.  Requests of kBigBlock bytes or more are first
// served from a per-device cache of IDLE large blocks (best fit, never split) that freed spaces
// leave behind: a build + solve of the same instance then re-uses exactly the blocks of the
// previous one instead of depending on the pool's (fragmenting) free lists.  `*got` = bytes.
constexpr size_t kBigBlock = size_t(16) << 20;
void* dev_alloc(size_t bytes, cudaStream_t s, size_t* got);
size_t device_bytes(int device); // total device memory (cached per device)
// Give back a block no pending work uses (its stream was synchronised): big blocks go to the
// cache (bounded; the oldest are freed past the bound), others to the pool on stream `s`.
void dev_release_idle(void* p, size_t bytes, cudaStream_t s);

// RAII device buffer on the stream-ordered allocator (cudaFreeAsync on the owner's stream),
// growable with copy.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0; // capacity in elements
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        n = 0;
    }
    // The owner's stream is synchronised: hand the block to the big-block cache.
    void release_idle() {
        if (p) dev_release_idle(p, n * sizeof(T), st);
        p = nullptr;
        n = 0;
    }
    // Ensure capacity >= want; keeps the first `keep` elements when it must reallocate.
    void reserve(size_t want, size_t keep, cudaStream_t s, double growth = 2.0) {
        if (want <= n) return;
        size_t cap = n ? static_cast<size_t>(static_cast<double>(n) * growth) : want;
        if (cap < want) cap = want;
        size_t got = 0;
        T* np = static_cast<T*>(dev_alloc(cap * sizeof(T), s, &got));
        if (p && keep)
            VCS_CUDA(cudaMemcpyAsync(np, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p) VCS_CUDA(cudaFreeAsync(p, s));
        p = np;
        n = got / sizeof(T);
        st = s;
    }
    // Discard contents; capacity >= `want` (grows geometrically to amortise re-allocation).
    void exact(size_t want, cudaStream_t s) {
        if (want <= n) return;
        const size_t cap = std::max<size_t>(want ? want : 1, n + n / 2);
        if (p) VCS_CUDA(cudaFreeAsync(p, s));
        p = nullptr;
        n = 0; // stays empty if the allocation below throws
        size_t got = 0;
        p = static_cast<T*>(dev_alloc(cap * sizeof(T), s, &got));
        n = got / sizeof(T);
        st = s;
    }
};

// Device-side control block of one solve.
struct SolveCtrl {
    int32_t stop;      // sticky: set by the first sweep that sees delta[k-1] < eps
    int32_t sweeps;    // K*: the converged sweep count
    int32_t certified; // certified pass: K* = H+1 proven, the wavefront fallback was skipped
    int32_t pad;
};

constexpr int kMethodAuto = 0;
constexpr int kMethodJacobi = 1;
constexpr int kMethodWavefront = 2;
constexpr int kMethodCertified = 3;

struct GraphKey {
    double eps;
    double discount;
    int skip;
    int max_sweeps;
    int method;
    int stream_out; // wavefront: record an event per layer (vcs_solve's overlapped download)
    bool operator<(const GraphKey& o) const {
        return std::tie(eps, discount, skip, max_sweeps, method, stream_out) <
               std::tie(o.eps, o.discount, o.skip, o.max_sweeps, o.method, o.stream_out);
    }
};

struct CachedGraph {
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> layer_ev; // wavefront + stream_out: after layer t's kernel
    int n_sweeps = 0; // sweep kernels in the graph
    int launches = 0;
    int method = kMethodJacobi;
    int uses = 0; // solves enqueued so far (the first runs without a graph)
    bool implicit = false; // certified pass on the implicit-CSR form: fallback runs at collect
    bool fallback_at_collect = false; // the proof's fallback is not in the graph (implicit / multi-GPU)
    int n_ranks = 1;       // GPUs (ranks) the solve ran on
};

struct MultiState;               // multi-GPU certified pass (vcs_solve.cu)
void destroy_multi(MultiState*); // waits for and frees everything it owns
struct CertShard;                // one rank of its multi-process form (vcs_cert_shard_*)
void destroy_cert_shard(CertShard*);

} // namespace vcs

struct vcs_space {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t d2h_stream = nullptr; // result copies overlapped with the layer pass
    cudaEvent_t order_ev = nullptr;    // a caller's solve stream waits for `stream` on it
    uint64_t S = 0, E = 0;
    int H = 0;
    int max_degree = 1;
    uint64_t max_layer = 0;
    double build_ms = 0.0;
    std::vector<uint64_t> layer_off;   // H+2
    std::vector<uint64_t> layer_edges; // H+1: edges leaving layer t
    bool has_plan = false;
    vcs::LayerPlan plan;
    std::vector<uint64_t> key_off;     // H+2: offset (u64 words) of layer t's packed keys

    // CSR in HBM (row_ptr u32 since E < 2^32 is enforced; succ u32 as mdp.hpp:126)
    vcs::DevBuf<uint32_t> row_ptr;
    vcs::DevBuf<uint32_t> succ;
    vcs::DevBuf<double> reward;
    vcs::DevBuf<int32_t> action;
    vcs::DevBuf<uint64_t> keys;
    // implicit-CSR form of a dense space (the persistent builder without EXPLICIT): the edges of
    // a state follow from its key and the layer's LayerParam; successor indices from the rank
    // tables.  The explicit CSR above is materialised on first use (vcs::ensure_csr).
    bool implicit = false;
    bool csr_ready = true;
    uint64_t state_cap = 0;
    vcs::DevBuf<uint32_t> rank_tables;  // per transition t at rank_off[t]
    std::vector<uint64_t> rank_off;     // H+1
    vcs::DevBuf<vcs::LayerParam> params_dev; // plan.layers on the device

    // value iteration state
    vcs::DevBuf<double> v[2];
    vcs::DevBuf<double> delta;   // residual per sweep (index k = sweep k)
    vcs::DevBuf<vcs::SolveCtrl> ctrl;
    vcs::DevBuf<int32_t> actions_dev;
    vcs::DevBuf<int8_t> act8_dev;          // int8 action column for the narrowed download
    std::vector<cudaEvent_t> piece_ev;     // events of the narrowed download pieces
    // layer-wavefront solver: version vectors of every layer + offsets
    vcs::DevBuf<double> ver;
    vcs::DevBuf<uint64_t> ver_off;
    vcs::DevBuf<uint64_t> layer_off_dev;
    std::vector<uint64_t> ver_off_host;
    // certified pass: (V_{m-1}, V_m) of every state, lower bounds lb[k] of the residuals
    vcs::DevBuf<double2> cert_xd;
    vcs::DevBuf<int8_t> cert_act_ks; // (VCS_CERT_PERMUTE) winner slots by key-space index
    vcs::DevBuf<unsigned char> stream_meta; // k_cert_stream's per-layer table
    vcs::DevBuf<uint32_t> stream_sync;      // its tile flags, layer counters, work counter
    uint32_t stream_tiles = 0;
    vcs::DevBuf<uint64_t> cert_tail_meta;   // k_cert_tail: row0 / n / key offset of layers 0..t
    int cert_tail_t = -1;
    bool cert_tail_ready = false;
    vcs::DevBuf<double> cert_lb;
    vcs::DevBuf<unsigned long long> cert_tl; // (VCS_CERT_TIMELINE) per-layer timeline stamps
    cudaStream_t aux_stream = nullptr; // captures the fallback body of the certified graph
    std::map<vcs::GraphKey, vcs::CachedGraph> graphs;
    vcs::CachedGraph* last_graph = nullptr; // graph of the last vcs_solve_enqueue
    vcs_solve_opts last_opts{};             // its options (the implicit-certified fallback)
    int last_key_skip = 1;
    // version-band sharded wavefront (vcs_wave_shard_*): this rank's band per layer
    int wave_world = 0, wave_rank = 0;
    double wave_eps = 1e-6, wave_discount = 1.0;
    std::vector<int> band_lo, band_hi, band_base, band_stride; // per layer 0..H
    std::vector<uint64_t> band_off;                             // per layer 0..H+1 (doubles)
    vcs::DevBuf<double> band_ver;                               // the rank's band store
    double* wave_delta = nullptr;                               // caller-owned residuals (H+3)
    double* shard_v0 = nullptr; // caller-owned device buffers of the sharded driver
    double* shard_v1 = nullptr;
    double* shard_delta = nullptr;
    int shard_n_delta = 0;

    // lazily built device index for locate (hash over (layer, key) -> state)
    vcs::DevBuf<uint32_t> loc_table;
    // results of the last collected solve (device-resident): vcs_policy_query reads them
    const double* result_values = nullptr;
    const int32_t* result_actions = nullptr;
    vcs::DevBuf<unsigned char> query_meta; // per layer: key layout for device-side packing
    uint64_t loc_cap = 0;

    int num_sms = 148;
    vcs::MultiState* multi = nullptr; // the multi-GPU solve's per-rank state (vcs_solve_multi)
    vcs::CertShard* cert_shard = nullptr; // vcs_cert_shard_* state of this process's rank
    uint64_t result_gen = 0;          // bumped whenever result_values / result_actions change
    // one caller at a time per space (the reference's const StateSpace may be shared by threads:
    // the solve, query and rollout entry points serialise on this)
    std::recursive_mutex mu;
    // caller streams that have run work on this space: the destructor waits for their last
    // recorded use before the space's blocks can be reused
    std::map<cudaStream_t, cudaEvent_t> use_ev;
    ~vcs_space();
};

namespace vcs {
// The stream an entry point enqueues on (the caller's, or the space's own when null).  On scope
// exit it records the caller stream's progress so vcs_space_free can wait for it.
struct StreamUse {
    vcs_space* sp;
    cudaStream_t s;
    StreamUse(vcs_space* space, void* stream)
        : sp(space), s(stream ? static_cast<cudaStream_t>(stream) : space->stream) {}
    StreamUse(const StreamUse&) = delete;
    StreamUse& operator=(const StreamUse&) = delete;
    ~StreamUse() {
        if (s == sp->stream) return;
        cudaEvent_t& ev = sp->use_ev[s];
        if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
            ev = nullptr;
            cudaStreamSynchronize(s); // cannot track it: finish it now
            return;
        }
        cudaEventRecord(ev, s);
    }
    operator cudaStream_t() const { return s; }
};
} // namespace vcs

namespace vcs {
bool trace_enabled(); // VCS_TRACE set: host-side phase timings on stderr
void ensure_csr(vcs_space* sp); // materialise the explicit CSR of an implicit space
double host_ms();
void bind_device(int device);
int sm_count(int device);
// Streams and events recycled across spaces on the current device (creating and destroying them
// costs tens of µs each: more than a tiny space's whole solve).  Released handles must be idle.
cudaStream_t acquire_stream(int device);
void release_stream(int device, cudaStream_t s);
cudaEvent_t acquire_event(int device, bool timing);
void release_event(int device, cudaEvent_t e, bool timing);
}
