// plan.cuh — a ptychography problem level resident on one device.
//
// Owns everything the hot path reads (positions, probe, amplitudes sqrt(d),
// optional raw intensities) and the scratch it writes (per-pattern stash,
// misfit partials, tile lists of the deterministic overlap-add).  Replaces
// the reference's ScanGeometry + DiffractionStack + Objective bundle
// (field.hpp:75-85, forward.hpp:22-27, objectives.hpp:18-26).
#pragma once

#include <memory>
#include <vector>

#include "blas.cuh"
#include "common.cuh"

namespace ptg {

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void alloc(size_t b) {
        release();
        if (b) PTG_CUDA(cudaMalloc(&p, b));
        bytes = b;
    }
    void ensure(size_t b) { if (bytes < b) alloc(b); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class X> X* as() const { return static_cast<X*>(p); }
};

struct HostPinned {
    void* p = nullptr;
    size_t bytes = 0;
    HostPinned() = default;
    HostPinned(const HostPinned&) = delete;
    HostPinned& operator=(const HostPinned&) = delete;
    ~HostPinned() { if (p) cudaFreeHost(p); }
    void ensure(size_t b) {
        if (bytes >= b) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        PTG_CUDA(cudaMallocHost(&p, b));
        bytes = b;
    }
    template <class X> X* as() const { return static_cast<X*>(p); }
};

// Patterns are processed in chunks whose stash fits the budget; each chunk
// carries the CSR lists of the object tiles its windows touch.
struct Chunk {
    int first = 0, count = 0;
    int ntiles = 0;          // tiles this chunk's gather visits
    bool all_tiles = false;  // single-chunk plans visit every tile (tile id = block id)
    int cap = 0;             // fixed stride of the per-tile window lists
    DevMem tile_ids, tile_list;
};

constexpr int kTileW = 64;   // overlap-add gather tile: 64 x 8 pixels, 2 per thread (32 x 8 block)
constexpr int kTileH = 8;
constexpr int kHvalDoubles = 16;
constexpr int kRmwInitBlocks = 1024;   // fixed grid of k_rmw_init => fixed <v,z> partition   // pinned host scalars per plan (never reallocated)

struct Comm;   // comm.cu (NCCL)

// Multi-GPU sharding of one problem (comm.cu, ptg_plan_create_sharded): this
// rank's positions are the contiguous scan block [pos_begin, pos_end) of the
// global scan; REPLICATED plans hold the whole object, BANDS plans object
// rows [row0, row0 + rows) = own_rows rows of their own + the halo their
// windows reach into the next rank's rows.
struct Shard {
    int layout = PTG_SHARD_NONE;
    int world = 1, rank = 0;
    int row0 = 0, own_rows = 0, halo_prev = 0;   // halo_prev: rows the previous rank's halo adds here
    int pos_begin = 0, pos_end = 0;
};

struct Plan {
    int n = 0, M = 0, w = 0, N = 0, prec = PTG_C64, device = 0;
    int rows = 0;                    // object rows held (n unless a BANDS shard)
    Shard shard;
    Comm* comm = nullptr;            // bound NCCL communicator (not owned)
    DevMem halo_buf;
    bool has_probe = false;
    std::vector<int32_t> pos_h;      // N x 2
    std::vector<double> probe_h;     // M x M complex128 (empty if binary)

    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    // banded host evaluation (plan_eval_host): copy-in / copy-out streams + events
    cudaStream_t s_in = nullptr, s_out = nullptr, s_in2 = nullptr, s_out2 = nullptr;
    // solver graphs: side stream + fork/join events (d_lbfgs products)
    cudaStream_t s_side = nullptr;
    cudaEvent_t ev_side[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_band;
    DevMem stage_out;
    // the banded host evaluation replayed as one CUDA graph (pinned host
    // buffers): keyed on every pointer the captured sequence bakes in; the
    // first call with a key runs eagerly, the second captures
    struct HostGraph {
        cudaGraphExec_t exec = nullptr;
        std::vector<const void*> key, seen;
        int64_t launches = 0;   // kernels per replay (launch accounting)
    } hg;

    DevMem pos, probe;
    DevMem probe_epi;                // complex64 TMA path: sc * P per metric (2 x M x M), sc = 1/M^2 | 2
    DevMem amp, inten;               // sqrt(d) and d, real type of the precision
    bool amp_valid = false, inten_valid = false;

    DevMem stash, misfit, dotp, value, scratch, flag, frame;
    DevMem counter;                  // last-block-done counter of the fused gather
    DevMem zbuf, vbuf, gbuf, stage;  // host-API working buffers
    HostPinned hval;   // kHvalDoubles, allocated once at plan creation

    // opt-in event timing of the frame kernel / gather (ptg_plan_set_timing)
    struct EvPair { cudaEvent_t a = nullptr, b = nullptr; int kind = 0; };
    bool timing = false;
    std::vector<EvPair> ev_pool;
    size_t ev_used = 0;
    void ev_begin(int kind);
    void ev_end();
    void timing_collect(double* ms, int64_t* cnt);   // ms[2], cnt[2]

    // TMA tensor maps (opaque 128-B CUtensorMap blobs) for the complex64 fast path
    alignas(64) unsigned char tm_amp[128] = {};
    const void* tm_amp_ptr = nullptr;
    alignas(64) unsigned char tm_probe[128] = {};
    bool tm_probe_ok = false;
    alignas(64) unsigned char tm_probe_epi[2][128] = {};   // maps of probe_epi (one per metric)
    struct TmEntry { const void* ptr = nullptr; alignas(64) unsigned char map[128] = {}; };
    std::vector<TmEntry> tm_z_cache = std::vector<TmEntry>(8);
    size_t tm_z_next = 0;

    // Overlap-add mode.  PLANES: scan positions are coloured into sets of
    // pairwise non-overlapping windows; each frame stores its contribution
    // into its colour's n x n plane (plain stores, disjoint within a colour)
    // and a streaming kernel sums the planes in fixed colour order.  STASH:
    // per-position contributions + tile-list gather (large problems).
    bool planes_mode = false;
    int ncolors = 0;
    std::vector<int> color_h;
    DevMem color, planes;

    // cluster-split objective kernel for complex64 M = 128 / 256 (frame_cl.cuh):
    // amplitudes permuted into its frequency order, rebuilt when the source
    // buffer or the data generation changes
    bool cl = false;
    DevMem amp_cl, cl_tw;
    const void* amp_cl_src = nullptr;
    int amp_cl_line = 0;
    uint64_t amp_cl_gen = ~0ull;
    uint64_t data_gen = 0;   // bumped whenever amp / inten are rewritten

    // RMW overlap-add (frame_rmw.cuh): persistent cluster kernel adding each
    // frame's contribution straight into the gradient in a fixed,
    // dependency-ordered sequence (no stash, no gather)
    bool rmw_mode = false;
    int rmw_clusters = 0;            // persistent grid (co-resident clusters)
    DevMem rmw_order, rmw_dep_off, rmw_dep_idx, rmw_done, rmw_work;
    std::vector<int> rmw_order_h;    // for tests / diagnostics
    // row groups of the order (ascending window rows): end index and largest
    // window row of each; suffix minimum of the window rows (banded host eval)
    std::vector<int> rmw_group_end, rmw_group_maxr0, rmw_sufmin_r0;

    // multi-pass path for frames larger than one CTA (frame_multipass.cuh)
    bool mp = false;
    int mp_chunk = 0;                // positions per scratch sub-chunk
    DevMem mp_scratch;               // mp_chunk x M x M complex
    int misfit_per_pos = 1;          // partial objective values per position

    int tiles_x = 0, tiles_y = 0;
    int chunk_size = 0;
    std::vector<std::unique_ptr<Chunk>> chunks;
    int64_t launches = 0;
    // the complex64 TMA frame kernel is launched with programmatic dependent
    // launch (set by the solvers while they capture their iteration graphs;
    // never for a timed standalone evaluation)
    bool pdl_frames = false;

    ~Plan();
    size_t celem() const { return prec == PTG_C64 ? 8 : 16; }
    size_t relem() const { return prec == PTG_C64 ? 4 : 8; }
    size_t nn() const { return (size_t)rows * n; }   // object elements held (rows x n)
    size_t MM() const { return (size_t)M * M; }
    bool ref_mode() const { return !has_probe && M == n; }
    size_t device_bytes() const;
};

// RAII: route blas/transfer launch counting into a plan
struct LaunchScope {
    int64_t* prev;
    explicit LaunchScope(Plan& p) : prev(g_launch_counter) { g_launch_counter = &p.launches; }
    ~LaunchScope() { g_launch_counter = prev; }
};

std::unique_ptr<Plan> plan_create(const ptg_plan_desc& d);
// this rank's share of a global problem (layout PTG_SHARD_REPLICATED | BANDS)
std::unique_ptr<Plan> plan_create_sharded(const ptg_plan_desc& global, int world, int rank, int layout);
// the partition itself (host only): out = {pos_begin, pos_end, row0, rows, own_rows, halo_prev}
void shard_layout(int n, int w, int N, const int32_t* positions, int world, int rank, int layout, int out[6]);
// NCCL (comm.cu)
void comm_unique_id(unsigned char out[128]);
Comm* comm_init(const unsigned char id[128], int world, int rank, int device);
void comm_destroy(Comm* c);
int comm_world(const Comm* c);
int comm_rank(const Comm* c);
void comm_exchange(Plan& p, void* grad, double* value_dev);   // after the local frames
void comm_sync_halo(Plan& p, void* z);                        // BANDS: z's halo rows from rank + 1
// status 4 unless `device` is a usable sm_100 device (selects it)
void check_device_public(int device);
// coarse plan built on device from a fine one (patch-model coarsening)
std::unique_ptr<Plan> plan_coarsen(Plan& fine);
void plan_set_data_host(Plan& p, const void* data, int dtype);
void plan_set_data_device(Plan& p, const void* data, int dtype);
void plan_load_ptyf(Plan& p, const char* path);   // PTYF stack file, streamed upload
void plan_ensure(Plan& p, int metric);   // make amp / inten valid for metric
// intensities rewritten on device: d >= 0 check + amplitudes (checkPattern)
void plan_refresh_amp(Plan& p);
// addNoise (forward.cpp:56-86) in place on the plan's data; uniforms_host =
// NULL draws Philox4x64-10 (seed), else 2 N M^2 uniforms in the reference's order
void plan_add_noise(Plan& p, double level, unsigned long long seed, const double* uniforms_host);
// Poisson photon noise at `photons` per pattern (counter-based, seed)
void plan_add_poisson(Plan& p, double photons, unsigned long long seed);
// raw Philox4x64-10 blocks: out[4 b + k] = philox(ctr + (b, 0, 0, 0), key)[k]
void dev_philox_raw(unsigned long long* out, size_t nblocks, const unsigned long long ctr[4],
                    const unsigned long long key[2], cudaStream_t s);

// objective + gradient on device buffers (plan precision); grad may be null
void plan_eval(Plan& p, int metric, const void* z, const void* v, void* grad, double* value_dev);
// the same from / to host complex128 buffers (ptg_eval); banded so that the
// PCIe copies of z in and the gradient out overlap the computation
void plan_eval_host(Plan& p, int metric, const double* z, const double* v, double* value, double* grad);
void plan_simulate(Plan& p, const void* z);
void plan_project(Plan& p, const void* z, int k, void* frame_out);
// fft2 / ifft2 of a device n x n complex128 field (synchronises s)
void dev_fft2(const void* in, int n, bool inverse, void* out, cudaStream_t s);
// one PIE sweep in place on device object z
void plan_pie_sweep(Plan& p, void* z, double gamma);

// host helpers
void plan_upload_c128(Plan& p, const double* host, void* dev);   // host c128 -> device prec
void plan_download_c128(Plan& p, const void* dev, double* host);
double plan_read_scalar(Plan& p, const double* dev);              // synchronising read
bool plan_nonfinite(Plan& p, const void* x, size_t len);
double plan_dot(Plan& p, const void* a, const void* b, size_t len);   // synchronising

}  // namespace ptg
