// plan.cu — device-resident problem + the objective/gradient pipeline.
//
// plan_eval restates evaluate/phiDistance/phiIntensityGaussian
// (/root/reference/proj/src/objectives.cpp:52-118) as, per pattern chunk:
//   1. frame_kernel<OP>   one CTA per scan position: gather, 2-D FFT, spectral
//                         misfit (fp64 block reduction), inverse FFT, conj(P)
//                         epilogue -> stash[j] (w x w)
//   2. k_overlap_gather   one CTA per 32x32 object tile: sums the stashes of
//                         the windows covering the tile in ascending scan
//                         order (the reference's accumulation order,
//                         objectives.cpp:59-72), subtracts the shift v and
//                         reduces <v,z>_R per tile — deterministic, no atomics
//   3. k_finalize         value = sum_j misfit_j - sum_t dot_t (fixed tree)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>

#include <cudaTypedefs.h>

#include "frame_cl.cuh"
#include "frame_rmw.cuh"
#include "frame_rmw2.cuh"
#include "frame_sc.cuh"
#include "frame_kernels.cuh"
#include "frame_multipass.cuh"
#include "frame_tma.cuh"
#include "pie_reg.cuh"
#include "plan.cuh"
#include "transfer.cuh"

namespace ptg {

Plan::~Plan() {
    for (auto& e : ev_pool) {
        if (e.a) cudaEventDestroy(e.a);
        if (e.b) cudaEventDestroy(e.b);
    }
    if (hg.exec) cudaGraphExecDestroy(hg.exec);
    for (auto e : ev_band) cudaEventDestroy(e);
    if (ev_side[0]) cudaEventDestroy(ev_side[0]);
    if (ev_side[1]) cudaEventDestroy(ev_side[1]);
    if (s_side) cudaStreamDestroy(s_side);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (s_in2) cudaStreamDestroy(s_in2);
    if (s_out2) cudaStreamDestroy(s_out2);
    if (own_stream) cudaStreamDestroy(own_stream);
}

void Plan::ev_begin(int kind) {
    if (!timing) return;
    if (ev_used == ev_pool.size()) {
        EvPair e;
        PTG_CUDA(cudaEventCreate(&e.a));
        PTG_CUDA(cudaEventCreate(&e.b));
        ev_pool.push_back(e);
    }
    ev_pool[ev_used].kind = kind;
    PTG_CUDA(cudaEventRecord(ev_pool[ev_used].a, stream));
}

void Plan::ev_end() {
    if (!timing) return;
    PTG_CUDA(cudaEventRecord(ev_pool[ev_used].b, stream));
    ++ev_used;
}

void Plan::timing_collect(double* ms, int64_t* cnt) {   // ms[3], cnt[3] (kind 2 = probes)
    ms[0] = ms[1] = ms[2] = 0.0;
    cnt[0] = cnt[1] = cnt[2] = 0;
    for (size_t i = 0; i < ev_used; ++i) {
        PTG_CUDA(cudaEventSynchronize(ev_pool[i].b));
        float t = 0.f;
        PTG_CUDA(cudaEventElapsedTime(&t, ev_pool[i].a, ev_pool[i].b));
        ms[ev_pool[i].kind] += t;
        cnt[ev_pool[i].kind] += 1;
    }
    ev_used = 0;
}

size_t Plan::device_bytes() const {
    size_t b = pos.bytes + probe.bytes + amp.bytes + inten.bytes + stash.bytes + misfit.bytes +
               dotp.bytes + value.bytes + scratch.bytes + flag.bytes + frame.bytes + zbuf.bytes +
               vbuf.bytes + gbuf.bytes + stage.bytes;
    for (const auto& c : chunks) b += c->tile_ids.bytes + c->tile_list.bytes;
    return b;
}

namespace {

// ------------------------------------------------------------ frame launch
template <int M>
constexpr int frame_threads() {
    return M <= 8 ? 32 : M == 16 ? 64 : M == 32 ? 128 : M == 64 ? 256 : 512;
}

// opt-in dynamic shared memory above 48 KB, once per kernel and device (the
// attribute is per device; one process may drive plans on several devices)
template <class K>
void set_smem_attr(K kern, size_t smem) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;   // (kernel, device)
    int dev = 0;
    PTG_CUDA(cudaGetDevice(&dev));
    const std::pair<const void*, int> key{reinterpret_cast<const void*>(kern), dev};
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return;
    PTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done.insert(key);
}

template <typename T, int M, int OP>
void launch_frame_t(const FrameArgs<T>& a, int count, cudaStream_t s) {
    constexpr int NT = frame_threads<M>();
    const size_t smem = frame_smem_bytes<T, M>(NT);
    auto kern = frame_kernel<T, M, NT, OP>;
    set_smem_attr(kern, smem);
    kern<<<count, NT, smem, s>>>(a);
    PTG_CHECK_LAUNCH();
}

template <typename T, int OP>
void launch_frame_m(int M, const FrameArgs<T>& a, int count, cudaStream_t s) {
    switch (M) {
        case 1: launch_frame_t<T, 1, OP>(a, count, s); break;
        case 2: launch_frame_t<T, 2, OP>(a, count, s); break;
        case 4: launch_frame_t<T, 4, OP>(a, count, s); break;
        case 8: launch_frame_t<T, 8, OP>(a, count, s); break;
        case 16: launch_frame_t<T, 16, OP>(a, count, s); break;
        case 32: launch_frame_t<T, 32, OP>(a, count, s); break;
        case 64: launch_frame_t<T, 64, OP>(a, count, s); break;
        case 128:
            if constexpr (sizeof(T) == 4) {
                launch_frame_t<T, 128, OP>(a, count, s);
                break;
            }
            [[fallthrough]];
        default:
            raise(PTG_ERR_CONFIG, "frame side M=" + std::to_string(M) +
                                      " exceeds the single-CTA shared-memory path for this precision");
    }
}

// ---------------------------------------------- TMA tensor maps (driver API)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        PTG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) raise(PTG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// n x n complex64 viewed as float32 [n][2n]; box = M rows x (M + extra) complex
// (the object window uses extra = 2 so its start can be rounded down to an even
// column: TMA box starts must be 16-B aligned)
void encode_z(CUtensorMap* tm, const void* z, int n, int M, int extra) {
    cuuint64_t dims[2] = {(cuuint64_t)2 * n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)2 * n * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)(2 * (M + extra)), (cuuint32_t)M};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(z), dims, strides,
                             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(PTG_ERR_CUDA, "tensor map (object) encode failed: " + std::to_string((int)r));
}

// amplitudes float32 [N][M][M]; box = (min(M,32) x M) tile of one pattern, swizzled
void encode_amp(CUtensorMap* tm, const void* amp, int M, int N) {
    const int AT = M < 32 ? M : 32;
    cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)M, (cuuint64_t)N};
    cuuint64_t strides[2] = {(cuuint64_t)M * sizeof(float), (cuuint64_t)M * M * sizeof(float)};
    cuuint32_t box[3] = {(cuuint32_t)AT, (cuuint32_t)M, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(amp), dims, strides,
                             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             AT == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(PTG_ERR_CUDA, "tensor map (data) encode failed: " + std::to_string((int)r));
}

// conj(sc * P) for the complex64 TMA epilogue
__global__ void k_scale_conj_c64(float2* __restrict__ out, const float2* __restrict__ in, float sc, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = make_float2(in[i].x * sc, -(in[i].y * sc));
}

// conj(sc * P) per metric (sc = 1/M^2 distance, 2 intensity: powers of two,
// so the table is exact), read by the complex64 epilogues: the contribution
// is then one packed complex multiply.  [0] distance, [1] intensity.
const float2* probe_epi_table(Plan& p, int op) {
    if (!p.probe_epi.p) {
        p.probe_epi.alloc(2 * p.MM() * sizeof(float2));
        float2* pe = p.probe_epi.as<float2>();
        const float sc[2] = {1.f / ((float)p.M * (float)p.M), 2.f};
        for (int k = 0; k < 2; ++k) {
            k_scale_conj_c64<<<(unsigned)((p.MM() + 255) / 256), 256, 0, p.stream>>>(
                pe + k * p.MM(), p.probe.as<const float2>(), sc[k], p.MM());
            PTG_CHECK_LAUNCH();
        }
    }
    return p.probe_epi.as<const float2>() + (op == OP_INTENSITY ? p.MM() : 0);
}

bool tma_path_ok(const Plan& p) {
    return p.prec == PTG_C64 && (p.M == 16 || p.M == 32 || p.M == 64) && p.w == p.M && p.n % 2 == 0 &&
           p.N > 0;
}

template <int M, int OP, bool PROBE>
void launch_tma_p(const FrameArgs<float>& a, int count, const CUtensorMap& tz, const CUtensorMap& ta,
                  const CUtensorMap& tp, cudaStream_t s, bool pdl) {
    constexpr int FPC = tma_frames_per_cta<M>();
    constexpr size_t smem = tma_smem_bytes<M>();
    auto kern = frame_tma_kernel<M, OP, PROBE>;
    set_smem_attr(kern, smem);
    if (!pdl) {
        kern<<<(count + FPC - 1) / FPC, M * FPC, smem, s>>>(a, count, tz, ta, tp);
    } else {   // solver graphs: launch (and the probe prefetch) overlap the predecessor
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((count + FPC - 1) / FPC);
        cfg.blockDim = dim3(M * FPC);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PTG_CUDA(cudaLaunchKernelEx(&cfg, kern, a, count, tz, ta, tp));
    }
    PTG_CHECK_LAUNCH();
}

template <int OP>
void launch_tma(Plan& p, const FrameArgs<float>& a, int count, const void* z, const float* data) {
    // cached maps: amplitudes per (buffer, metric); object per pointer (small LRU)
    if (p.tm_amp_ptr != data) {
        encode_amp(reinterpret_cast<CUtensorMap*>(p.tm_amp), data, p.M, p.N);
        p.tm_amp_ptr = data;
    }
    CUtensorMap* tz = nullptr;
    for (auto& e : p.tm_z_cache)
        if (e.ptr == z) tz = reinterpret_cast<CUtensorMap*>(e.map);
    if (!tz) {
        auto& e = p.tm_z_cache[p.tm_z_next++ % p.tm_z_cache.size()];
        encode_z(reinterpret_cast<CUtensorMap*>(e.map), z, p.n, p.M, 2);
        e.ptr = z;
        tz = reinterpret_cast<CUtensorMap*>(e.map);
    }
    const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(p.tm_amp);
    const bool pr = a.probe != nullptr;
    if (pr && !p.tm_probe_ok) {   // M x M complex64 as float32 [M][2M], one box
        const float2* pe = probe_epi_table(p, 0);
        for (int k = 0; k < 2; ++k)
            encode_z(reinterpret_cast<CUtensorMap*>(p.tm_probe_epi[k]), pe + k * p.MM(), p.M, p.M, 0);
        p.tm_probe_ok = true;
    }
    const CUtensorMap& tp =
        pr ? *reinterpret_cast<const CUtensorMap*>(p.tm_probe_epi[OP == OP_INTENSITY ? 1 : 0]) : *tz;
    switch (p.M) {
        case 16: pr ? launch_tma_p<16, OP, true>(a, count, *tz, ta, tp, p.stream, p.pdl_frames) : launch_tma_p<16, OP, false>(a, count, *tz, ta, tp, p.stream, p.pdl_frames); break;
        case 32: pr ? launch_tma_p<32, OP, true>(a, count, *tz, ta, tp, p.stream, p.pdl_frames) : launch_tma_p<32, OP, false>(a, count, *tz, ta, tp, p.stream, p.pdl_frames); break;
        default: pr ? launch_tma_p<64, OP, true>(a, count, *tz, ta, tp, p.stream, p.pdl_frames) : launch_tma_p<64, OP, false>(a, count, *tz, ta, tp, p.stream, p.pdl_frames); break;
    }
}

// ------------------------------------------- cluster-split frames (M = 128, 256)
bool cl_path_ok(const Plan& p) {
    static const bool off = getenv("PTG_NO_CLUSTER") && getenv("PTG_NO_CLUSTER")[0] == '1';   // A/B switch
    return !off && p.prec == PTG_C64 && (p.M == 128 || p.M == 256) && p.w == p.M && p.N > 0;
}

// local line length of the cluster kernel: M = Q L with L = 32 (default:
// twice the CTAs per SM) or 64 (PTG_CL_L=64, A/B)
int cl_line(const Plan& p) {
    static const int env = getenv("PTG_CL_L") ? atoi(getenv("PTG_CL_L")) : 0;
    return env == 64 ? 64 : 32;
}
constexpr int kSplitLine = 33;   // cl_amp tag: the split (two threads per line) order of frame_rmw2_kernel
// PTG_RMW2=1: M = 256 RMW plans use frame_rmw2_kernel (512 threads, two per
// line: 46 % warps active instead of 23 %).  Measured and kept off by default:
// 24.7 vs 22.1 ms per config-5 evaluation -- barrier (26 %) and MIO-throttle
// (21 %) stalls grow with the extra shared-memory reads of the split lines
bool rmw2(const Plan& p) {
    if (p.M != 256) return false;
    const char* e = getenv("PTG_RMW2");
    return e && e[0] == '1';
}
// local line of the persistent RMW kernel: 8-CTA (M = 256) / 4-CTA (M = 128)
// clusters of 32-row CTAs.  Measured and rejected: 16-CTA clusters of 16-row
// CTAs at 3 per SM (M = 256): 27.9 vs 22.5 ms per config-5 evaluation (more
// cluster-barrier and membar stalls, 25 % more instructions)
int rmw_line(const Plan&) { return 32; }

template <int Q, int L>
void perm_amp(Plan& p, const float* data, size_t total) {
    const int grid = (int)std::min<size_t>(148 * 16, (total + 255) / 256);
    k_perm_amp<Q, L><<<grid, 256, 0, p.stream>>>(data, p.amp_cl.as<float>(), total);
    PTG_CHECK_LAUNCH();
    ++p.launches;
}

// amplitudes (or intensities) permuted for frame_cl_kernel, rebuilt when the
// source buffer, its contents (data_gen) or the split change
const float* cl_amp(Plan& p, const float* data, int L) {
    if (p.amp_cl_src != data || p.amp_cl_gen != p.data_gen || p.amp_cl_line != L) {
        const size_t total = (size_t)p.N * p.MM();
        p.amp_cl.ensure(total * sizeof(float));
        if (L == kSplitLine) {   // frame_rmw2_kernel's order (M = 256)
            const int grid = (int)std::min<size_t>(148 * 16, (total + 255) / 256);
            k_perm_amp_split<<<grid, 256, 0, p.stream>>>(data, p.amp_cl.as<float>(), total);
            PTG_CHECK_LAUNCH();
            ++p.launches;
        } else if (p.M == 128) {
            L == 32 ? perm_amp<4, 32>(p, data, total) : perm_amp<2, 64>(p, data, total);
        } else {
            L == 32 ? perm_amp<8, 32>(p, data, total) : perm_amp<4, 64>(p, data, total);
        }
        p.amp_cl_src = data;
        p.amp_cl_gen = p.data_gen;
        p.amp_cl_line = L;
    }
    return p.amp_cl.as<const float>();
}

template <int Q, int L, int OP, bool PROBE>
void launch_cl_t(Plan& p, const FrameArgs<float>& a, int count, const float* amp_perm, const float2* tw) {
    constexpr size_t smem = cl_smem_bytes<Q, L>();
    auto kern = frame_cl_kernel<Q, L, OP, PROBE>;
    set_smem_attr(kern, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)count * Q);
    cfg.blockDim = dim3(Q * L);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = p.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = Q;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const float2* pe = PROBE ? probe_epi_table(p, OP) : nullptr;
    PTG_CUDA(cudaLaunchKernelEx(&cfg, kern, a, amp_perm, tw, pe));
}

template <int Q, int L, int OP>
void launch_cl_ql(Plan& p, const FrameArgs<float>& a, int count, const float* ap, const float2* tw) {
    if (a.probe) launch_cl_t<Q, L, OP, true>(p, a, count, ap, tw);
    else launch_cl_t<Q, L, OP, false>(p, a, count, ap, tw);
}

// W_M^i, i < M, in fp64 rounded once
const float2* cl_twiddles(Plan& p) {
    if (!p.cl_tw.p) {
        std::vector<float> h(2 * (size_t)p.M);
        for (int i = 0; i < p.M; ++i) {
            const double th = 2.0 * M_PI * i / p.M;
            h[2 * i] = (float)std::cos(th);
            h[2 * i + 1] = (float)-std::sin(th);
        }
        p.cl_tw.alloc(h.size() * sizeof(float));
        PTG_CUDA(cudaMemcpyAsync(p.cl_tw.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, p.stream));
    }
    return p.cl_tw.as<const float2>();
}

template <int OP>
void launch_cl(Plan& p, const FrameArgs<float>& a, int count, const float* data) {
    const float* ap = cl_amp(p, data, cl_line(p));
    const float2* tw = cl_twiddles(p);
    const int L = cl_line(p);
    if (p.M == 128) L == 32 ? launch_cl_ql<4, 32, OP>(p, a, count, ap, tw) : launch_cl_ql<2, 64, OP>(p, a, count, ap, tw);
    else L == 32 ? launch_cl_ql<8, 32, OP>(p, a, count, ap, tw) : launch_cl_ql<4, 64, OP>(p, a, count, ap, tw);
}

// ------------------------------------------- persistent RMW frames (M = 128, 256)
template <int Q, int L, int OP, bool PROBE>
void launch_rmw_t(Plan& p, const FrameArgs<float>& a, const float* amp_perm, const float2* tw, float2* grad,
                  int kbeg, int kend) {
    // PTG_RMW_SMEM_PAD=bytes (diagnostic): extra dynamic shared memory, e.g. to
    // force one CTA per SM and read off how much two co-resident frames overlap
    static const size_t pad = getenv("PTG_RMW_SMEM_PAD") ? (size_t)atoll(getenv("PTG_RMW_SMEM_PAD")) : 0;
    const size_t smem = cl_smem_bytes<Q, L>() + pad;
    // probe rows cached in tensor memory (frame_rmw.cuh): M = 256 probe frames
    constexpr bool TMC = PROBE && Q == 8;
    const char* etm = getenv("PTG_RMW_TMEM");   // A/B switch, read per launch
    const bool tm_off = etm && etm[0] == '0';
    const bool tm = TMC && !tm_off;
    auto kern_sizing = frame_rmw_kernel<Q, L, OP, PROBE, false>;   // occupancy query (see frame_rmw.cuh)
    auto kern = tm ? frame_rmw_kernel<Q, L, OP, PROBE, TMC> : kern_sizing;
    set_smem_attr(kern_sizing, smem);
    set_smem_attr(kern, smem);
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(Q * L);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = p.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = Q;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (!p.rmw_clusters) {   // persistent grid: the clusters that fit at once
        cfg.gridDim = dim3(Q);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void*)kern_sizing, &cfg) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            ncl = 148 / Q;
        }
        // PTG_RMW_CLUSTERS=C (diagnostic): override the persistent grid
        if (const char* e = getenv("PTG_RMW_CLUSTERS")) ncl = std::max(1, atoi(e));
        if (getenv("PTG_RMW_DEBUG")) fprintf(stderr, "[rmw] Q=%d L=%d: %d co-resident clusters, %zu B smem/CTA\n", Q, L, ncl, smem);
        p.rmw_clusters = ncl;
    }
    const int ncl = std::max(1, std::min(p.rmw_clusters, kend - kbeg));
    cfg.gridDim = dim3((unsigned)ncl * Q);
    RmwArgs r{p.rmw_order.as<const int>(), p.rmw_dep_off.as<const int>(), p.rmw_dep_idx.as<const int>(),
              p.rmw_done.as<unsigned>(), p.rmw_work.as<unsigned>(), grad, kbeg, kend};
    const float2* pe = PROBE ? probe_epi_table(p, OP) : nullptr;
    PTG_CUDA(cudaLaunchKernelEx(&cfg, kern, a, amp_perm, tw, pe, r));
}

template <int OP, bool PROBE>
void launch_rmw2_t(Plan& p, const FrameArgs<float>& a, const float* amp_perm, const float2* tw, float2* grad,
                   int kbeg, int kend) {
    constexpr size_t smem = cl_smem_bytes<8, 32>();
    auto kern = frame_rmw2_kernel<OP, PROBE>;
    set_smem_attr(kern, smem);
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = p.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (!p.rmw_clusters) {
        cfg.gridDim = dim3(8);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            ncl = 148 / 8;
        }
        p.rmw_clusters = ncl;
    }
    const int ncl = std::max(1, std::min(p.rmw_clusters, kend - kbeg));
    cfg.gridDim = dim3((unsigned)ncl * 8);
    RmwArgs r{p.rmw_order.as<const int>(), p.rmw_dep_off.as<const int>(), p.rmw_dep_idx.as<const int>(),
              p.rmw_done.as<unsigned>(), p.rmw_work.as<unsigned>(), grad, kbeg, kend};
    const float2* pe = PROBE ? probe_epi_table(p, OP) : nullptr;
    PTG_CUDA(cudaLaunchKernelEx(&cfg, kern, a, amp_perm, tw, pe, r));
}

// M = 128: the four-CTA cluster fused into one persistent 512-thread CTA per SM (frame_sc.cuh)
template <int OP, bool PROBE>
void launch_sc_t(Plan& p, const FrameArgs<float>& a, const float* amp_perm, const float2* tw, float2* grad, int kbeg,
                 int kend) {
    constexpr size_t smem = sc_smem_bytes();
    const char* etm = getenv("PTG_RMW_TMEM");   // A/B switch, read per launch
    const bool tm = PROBE && !(etm && etm[0] == '0');
    auto kern = tm ? frame_sc_kernel<OP, PROBE, PROBE> : frame_sc_kernel<OP, PROBE, false>;
    set_smem_attr(kern, smem);
    int sms = 0;
    PTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
    const int grid = std::max(1, std::min(sms, kend - kbeg));
    RmwArgs r{p.rmw_order.as<const int>(), p.rmw_dep_off.as<const int>(), p.rmw_dep_idx.as<const int>(),
              p.rmw_done.as<unsigned>(), p.rmw_work.as<unsigned>(), grad, kbeg, kend};
    const float2* pe = PROBE ? probe_epi_table(p, OP) : nullptr;
    kern<<<grid, kScThreads, smem, p.stream>>>(a, amp_perm, tw, pe, r);
    PTG_CHECK_LAUNCH();
}

// frames [kbeg, kend) of the RMW order; the dispatch counter must be zero
template <int OP>
void launch_rmw(Plan& p, const FrameArgs<float>& a, const float* data, float2* grad, int kbeg, int kend) {
    if (rmw2(p)) {
        const float* ap = cl_amp(p, data, kSplitLine);
        const float2* tw = cl_twiddles(p);
        a.probe ? launch_rmw2_t<OP, true>(p, a, ap, tw, grad, kbeg, kend)
                : launch_rmw2_t<OP, false>(p, a, ap, tw, grad, kbeg, kend);
        return;
    }
    const float* ap = cl_amp(p, data, rmw_line(p));
    const float2* tw = cl_twiddles(p);
    // PTG_ABL_NOPROBE=1: timing ablation only (the probe-free kernel on a
    // probe problem: wrong results), measures what the probe loads cost
    static const bool abl_noprobe = getenv("PTG_ABL_NOPROBE") && getenv("PTG_ABL_NOPROBE")[0] == '1';
    const bool probe = a.probe && !abl_noprobe;
    // PTG_SC=1 (A/B, read per launch): M = 128 frames by the fused 512-thread CTA (frame_sc.cuh)
    // instead of the four-CTA cluster -- bit-identical, measured slower (config 5's level 1, ms per
    // evaluation: fused 5.36 / cluster RMW 4.57 / stash 4.38; with PTG_RMW_SB=256 4.33 / 4.10)
    const char* esc = getenv("PTG_SC");
    const bool sc = esc && esc[0] == '1';
    if (p.M == 128 && sc)
        probe ? launch_sc_t<OP, true>(p, a, ap, tw, grad, kbeg, kend)
              : launch_sc_t<OP, false>(p, a, ap, tw, grad, kbeg, kend);
    else if (p.M == 128)
        probe ? launch_rmw_t<4, 32, OP, true>(p, a, ap, tw, grad, kbeg, kend)
              : launch_rmw_t<4, 32, OP, false>(p, a, ap, tw, grad, kbeg, kend);
    else
        probe ? launch_rmw_t<8, 32, OP, true>(p, a, ap, tw, grad, kbeg, kend)
              : launch_rmw_t<8, 32, OP, false>(p, a, ap, tw, grad, kbeg, kend);
}

// objective frame kernel: TMA/register path for complex64 patch frames up to
// M = 64, cluster-split register path for M = 128 / 256, smem path otherwise
template <typename T, int OP>
void launch_objective(Plan& p, const FrameArgs<T>& a, int count, const void* z, const T* data) {
    if constexpr (sizeof(T) == 4) {
        if (tma_path_ok(p)) {
            launch_tma<OP>(p, a, count, z, data);
            return;
        }
        if (p.cl) {
            launch_cl<OP>(p, a, count, data);
            return;
        }
    }
    launch_frame_m<T, OP>(p.M, a, count, p.stream);
}

// single-CTA frame kernels (whole frame in shared memory / registers)
bool frame_single_cta(int prec, int M) {
    return is_pow2(M) && (M <= 64 || (M == 128 && prec == PTG_C64));
}
bool frame_supported(int prec, int M) { return is_pow2(M) && M <= 512 && (frame_single_cta(prec, M) || M >= 128); }

// ------------------------------------------------------- multi-pass frames
template <typename T, int M, int OP>
void launch_mp_t(Plan& p, const FrameArgs<T>& a, int first, int count, int which) {
    constexpr size_t smem = mp_smem_bytes<T, M>();
    constexpr int NT = mp_threads<M>();
    set_smem_attr(mp_rows_fwd<T, M>, smem);
    set_smem_attr(mp_cols<T, M, OP>, smem);
    if constexpr (OP != OP_SIMULATE) set_smem_attr(mp_rows_inv<T, M, OP>, smem);
    MpArgs m{first, M / kMpLines, p.misfit.as<double>()};
    cplx<T>* scratch = p.mp_scratch.as<cplx<T>>();
    const dim3 grid(count, M / kMpLines);
    if (which & 1) { mp_rows_fwd<T, M><<<grid, NT, smem, p.stream>>>(a, m, scratch); PTG_CHECK_LAUNCH(); ++p.launches; }
    if (which & 2) { mp_cols<T, M, OP><<<grid, NT, smem, p.stream>>>(a, m, scratch); PTG_CHECK_LAUNCH(); ++p.launches; }
    if constexpr (OP != OP_SIMULATE) {
        if (which & 4) { mp_rows_inv<T, M, OP><<<grid, NT, smem, p.stream>>>(a, m, scratch); PTG_CHECK_LAUNCH(); ++p.launches; }
    }
}

// positions [first, first+count) through the three passes, in scratch-sized sub-chunks
template <typename T, int OP>
void launch_mp(Plan& p, const FrameArgs<T>& a, int first, int count, int which = 7) {
    for (int s = 0; s < count; s += p.mp_chunk) {
        const int cnt = std::min(p.mp_chunk, count - s);
        switch (p.M) {
            case 128: launch_mp_t<T, 128, OP>(p, a, first + s, cnt, which); break;
            case 256: launch_mp_t<T, 256, OP>(p, a, first + s, cnt, which); break;
            case 512: launch_mp_t<T, 512, OP>(p, a, first + s, cnt, which); break;
            default: raise(PTG_ERR_INTERNAL, "multi-pass frame size");
        }
    }
}

template <typename T>
FrameArgs<T> frame_args(Plan& p, const void* z, const T* amp) {
    FrameArgs<T> a{};
    a.z = static_cast<const cplx<T>*>(z);
    a.probe = p.has_probe ? p.probe.as<const cplx<T>>() : nullptr;
    a.pos = p.pos.as<const int2>();
    a.amp = amp;
    a.stash = p.stash.as<cplx<T>>();
    a.misfit = p.misfit.as<double>();
    a.planes = p.planes_mode ? p.planes.as<cplx<T>>() : nullptr;
    a.color = p.planes_mode ? p.color.as<const int>() : nullptr;
    a.n = p.n;
    a.w = p.w;
    return a;
}

__device__ __forceinline__ void finalize_block(const double* misfit, int N, const double* dotp, int ndot,
                                               double* out, double* red, int lin) {
    finalize_value<256>(misfit, N, dotp, ndot, out, red, lin);
}

// ------------------------------------------------------ colour-plane reduce
constexpr int kPlaneBlocks = 148 * 4;   // fixed grid => fixed dot partition (deterministic)
// grad = sum_c planes[c] (fixed colour order) - v, <v,z> partials, fused final
// value (last block).  Pure streaming: every thread owns a fixed pixel pair.
// QS lanes per pixel pair (small problems: more loads in flight per pair);
// lane q sums colours q, q + QS, ... in order, lanes combine by a fixed xor tree
template <typename T, int QS>
__global__ void __launch_bounds__(256, 4) k_plane_reduce(const cplx<T>* __restrict__ planes, int ncol, size_t nn,
                                                      const cplx<T>* __restrict__ v, const cplx<T>* __restrict__ z,
                                                      cplx<T>* __restrict__ grad, double* __restrict__ dotp,
                                                      const double* __restrict__ misfit, int N,
                                                      double* value_out, unsigned int* counter,
                                                      int block0) {
    // logical block b = block0 + blockIdx.x of a fixed kPlaneBlocks partition:
    // a launch may cover a subset of the blocks (banded host evaluation); the
    // fused final value (value_out) needs the full grid in one launch
    __shared__ double red[8];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lin = threadIdx.x;
    const int q = lin % QS;
    const unsigned gmask = QS == 1 ? 0u : (((1u << QS) - 1u) << ((lin & 31) & ~(QS - 1)));
    const int b = block0 + blockIdx.x;
    const size_t npairs = (nn + 1) / 2;
    const size_t chunk = (npairs + kPlaneBlocks - 1) / kPlaneBlocks;
    const size_t lo = min(npairs, b * chunk), hi = min(lo + chunk, npairs);
    if (!v && value_out && blockIdx.x == 0) {
        // no shift: every <v,z> partial is 0.0, so the value needs only the
        // misfits, final since griddepcontrol.wait -- block 0 forms it first
        // (same partition and order as the last-block path, bitwise equal),
        // overlapping the other blocks' plane reads, with no fence + counter
        // round trip anywhere
        finalize_block(misfit, N, dotp, 0, value_out, red, lin);
        __syncthreads();   // red[] is reused below
    }
    double d = 0.0;
    for (size_t pr = lo + lin / QS; pr < hi; pr += blockDim.x / QS) {
        const size_t i = 2 * pr;
        const bool two = i + 1 < nn;
        cplx<T> a0 = mk<T>(T(0), T(0)), a1 = a0;
        constexpr int B = 8;
        for (int c0 = q; c0 < ncol; c0 += B * QS) {
            cplx<T> q0[B], q1[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                q0[u] = q1[u] = mk<T>(T(0), T(0));
                if (c0 + u * QS < ncol) {
                    const cplx<T>* s = planes + (size_t)(c0 + u * QS) * nn + i;
                    if constexpr (sizeof(T) == 4) {
                        if (two && (nn % 2 == 0)) {   // 16-B aligned pair
                            const float4 f = __ldg(reinterpret_cast<const float4*>(s));
                            q0[u] = mk<T>(f.x, f.y);
                            q1[u] = mk<T>(f.z, f.w);
                        } else {
                            q0[u] = s[0];
                            if (two) q1[u] = s[1];
                        }
                    } else {
                        q0[u] = s[0];
                        if (two) q1[u] = s[1];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                a0 = cadd(a0, q0[u]);
                a1 = cadd(a1, q1[u]);
            }
        }
        if constexpr (QS > 1) {
#pragma unroll
            for (int o = 1; o < QS; o <<= 1) {
                a0 = cadd(a0, mk<T>(__shfl_xor_sync(gmask, a0.x, o), __shfl_xor_sync(gmask, a0.y, o)));
                a1 = cadd(a1, mk<T>(__shfl_xor_sync(gmask, a1.x, o), __shfl_xor_sync(gmask, a1.y, o)));
            }
            if (q != 0) continue;
        }
        if (v) {
            const cplx<T> v0 = v[i], z0 = z[i];
            a0 = csub(a0, v0);
            d += (double)v0.x * (double)z0.x + (double)v0.y * (double)z0.y;
            if (two) {
                const cplx<T> v1 = v[i + 1], z1 = z[i + 1];
                a1 = csub(a1, v1);
                d += (double)v1.x * (double)z1.x + (double)v1.y * (double)z1.y;
            }
        }
        grad[i] = a0;
        if (two) grad[i + 1] = a1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((lin & 31) == 0) red[lin >> 5] = d;
    __syncthreads();
    if (lin == 0) {
        double s = 0.0;
        for (int k = 0; k < 8; ++k) s += red[k];
        dotp[b] = s;
    }
    if (!value_out) return;   // partial launch: the value is formed by k_finalize
    if (!v) return;   // value formed by block 0 above
    __shared__ bool last;
    if (lin == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        finalize_block(misfit, N, dotp, gridDim.x, value_out, red, lin);
        if (lin == 0) *counter = 0u;
    }
}

// lanes per pixel pair of the plane reduce: the fixed partition gives each block
// `chunk` pairs; small planes (coarse MG levels) split a pair's colours over lanes
inline int plane_qs(const Plan& p) {
    const size_t chunk = ((p.nn() + 1) / 2 + kPlaneBlocks - 1) / kPlaneBlocks;
    return chunk <= 64 ? 4 : chunk <= 128 ? 2 : 1;
}
template <typename T>
auto plane_reduce_kernel(int qs) {
    return qs == 4 ? k_plane_reduce<T, 4> : qs == 2 ? k_plane_reduce<T, 2> : k_plane_reduce<T, 1>;
}

// --------------------------------------------------------- overlap gather
template <typename T>
__global__ void __launch_bounds__(256) k_overlap_gather(
    const cplx<T>* __restrict__ stash, const int* __restrict__ tile_ids,
    int cap, const int4* __restrict__ entries, int n, int w, int tiles_x,
    const cplx<T>* __restrict__ v,
    const cplx<T>* __restrict__ z, cplx<T>* __restrict__ grad, double* __restrict__ dotp,
    int accumulate, const double* __restrict__ misfit, int N, double* value_out,
    unsigned int* counter) {
    __shared__ double red[8];
    // programmatic dependent launch: everything above overlaps the frame
    // kernel's tail; wait here until its stash/misfit writes are visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int t = tile_ids ? tile_ids[blockIdx.x] : blockIdx.x;
    const int ty = t / tiles_x, tx = t % tiles_x;
    const int x = tx * kTileW + 2 * threadIdx.x;   // this lane's pixel pair (x, x+1), x even
    const int y = ty * kTileH + threadIdx.y;
    const int lin = threadIdx.y * 32 + threadIdx.x;
    const int sp = stash_pitch(w);
    // The tile's windows, in ascending scan order, are host-precomputed at a
    // fixed stride `cap` (padded with never-matching entries) as
    // {stash offset - r0*sp - even(c0), r0, even(c0)}.  Thanks to the stash
    // layout (parity-shifted, zero-padded rows of pitch w+2) a window touching
    // the pair contributes exactly one aligned 16-byte vector, zeros included:
    // one uniform entry load + one predicated vector load per window; the
    // adds follow the list (= the reference's accumulation order).
    constexpr int U = 16;
    cplx<T> a0 = mk<T>(T(0), T(0)), a1 = a0, v0 = a0, v1 = a0, z0 = a0, z1 = a0;
    const bool in0 = x < n && y < n, in1 = x + 1 < n && y < n;
    if (v) {   // shift operands prefetched off the critical path
        if (in0) { v0 = v[(size_t)y * n + x]; z0 = z[(size_t)y * n + x]; }
        if (in1) { v1 = v[(size_t)y * n + x + 1]; z1 = z[(size_t)y * n + x + 1]; }
    }
    const int pix = y * sp + x;
    // the block's entry list is staged once in shared memory: a warp-uniform
    // global LDG.128 would still move 512 B through the L1 data path per warp,
    // a broadcast LDS.128 costs one wavefront
    constexpr int LCAP = 256;
    __shared__ int4 s_e[LCAP];
    const int4* __restrict__ E = entries + (size_t)blockIdx.x * cap;
    for (int base = 0; base < cap; base += LCAP) {
    const int ccap = min(LCAP, cap - base);
    __syncthreads();
    for (int i = lin; i < ccap; i += 256) s_e[i] = __ldg(E + base + i);
    __syncthreads();
    for (int e = 0; e < ccap; e += U) {
        int4 en[U];
#pragma unroll
        for (int u = 0; u < U; ++u) en[u] = s_e[e + u];
        cplx<T> p0[U], p1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = (unsigned)(x - en[u].z) < (unsigned)(w + 2) && (unsigned)(y - en[u].y) < (unsigned)w;
            const cplx<T>* s = stash + (ok ? en[u].x + pix : 0);
            if constexpr (sizeof(T) == 4) {
                float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                if (ok) q = __ldg(reinterpret_cast<const float4*>(s));
                p0[u] = mk<T>(q.x, q.y);
                p1[u] = mk<T>(q.z, q.w);
            } else {
                p0[u] = ok ? s[0] : mk<T>(T(0), T(0));
                p1[u] = ok ? s[1] : mk<T>(T(0), T(0));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a0 = cadd(a0, p0[u]);
            a1 = cadd(a1, p1[u]);
        }
    }
    }
    double d = 0.0;
    cplx<T> g[2] = {a0, a1};
    const cplx<T> vv[2] = {v0, v1}, zz[2] = {z0, z1};
    const bool in[2] = {in0, in1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        if (!in[i]) continue;
        const size_t idx = (size_t)y * n + x + i;
        if (accumulate) g[i] = cadd(grad[idx], g[i]);
        if (v) {
            g[i] = csub(g[i], vv[i]);
            d += (double)vv[i].x * (double)zz[i].x + (double)vv[i].y * (double)zz[i].y;
        }
        grad[idx] = g[i];
    }
    if (v || value_out) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if ((lin & 31) == 0) red[lin >> 5] = d;
        __syncthreads();
        if (lin == 0) {
            double s = 0.0;
            for (int i = 0; i < 8; ++i) s += red[i];
            dotp[blockIdx.x] = s;
        }
    }
    if (value_out) {
        // fused finalize: the last block to finish reduces misfit + dot partials
        __shared__ bool last;
        if (lin == 0) {
            __threadfence();
            last = atomicAdd(counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            finalize_block(misfit, N, dotp, gridDim.x, value_out, red, lin);
            if (lin == 0) *counter = 0u;
        }
    }
}

// grad -= v ; dot partial per block (multi-chunk plans)
template <typename T>
__global__ void __launch_bounds__(256) k_shift(const cplx<T>* __restrict__ v, const cplx<T>* __restrict__ z,
                                               cplx<T>* __restrict__ grad, size_t len, double* dotp) {
    __shared__ double red[8];
    const size_t chunk = (len + gridDim.x - 1) / gridDim.x;
    const size_t lo = blockIdx.x * chunk, hi = min(lo + chunk, len);
    double d = 0.0;
    for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const cplx<T> vv = v[i], zz = z[i];
        grad[i] = csub(grad[i], vv);
        d += (double)vv.x * (double)zz.x + (double)vv.y * (double)zz.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < 8; ++i) s += red[i];
        dotp[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(256) k_finalize(const double* __restrict__ misfit, int N,
                                                  const double* __restrict__ dotp, int ndot,
                                                  double* __restrict__ out) {
    __shared__ double red[8];
    finalize_block(misfit, N, dotp, ndot, out, red, threadIdx.x);
}

// value -= sum of the dot partials (fixed order; one thread)
constexpr int kShiftBlocks = 1024;
__global__ void k_sub_dots(const double* __restrict__ dotp, int ndot, double* value) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int i = 0; i < ndot; ++i) s += dotp[i];
    *value -= s;
}

// --------------------------------------------------------------- data prep
// d >= 0 check (checkPattern, objectives.cpp:12-18) + amp = sqrt(d)
template <typename R>
__global__ void k_prepare(const R* __restrict__ d, size_t len, R* __restrict__ amp,
                          unsigned long long* bad) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const R x = d[i];
        if (x < R(0)) atomicMin(bad, (unsigned long long)i);
        amp[i] = sqrt(x);
    }
}

template <typename R>
__global__ void k_square(const R* __restrict__ a, size_t len, R* __restrict__ d) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        d[i] = a[i] * a[i];
}

inline int grid_for(size_t len) {
    size_t g = (len + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

// ------------------------------------------------------------------ PIE
// Strictly sequential sweep (solvers.cpp:244-251): one CTA walks the scan in
// order; each projection is a full smem 2-D FFT pair; z is updated in global
// memory and re-read (L2, __ldcg) by the next overlapping position.
template <typename T, int M, int NT>
__global__ void __launch_bounds__(NT) k_pie_sweep(cplx<T>* z, const cplx<T>* __restrict__ probe,
                                                  const int2* __restrict__ pos,
                                                  const T* __restrict__ amp, int N, int n, int w,
                                                  const cplx<T>* __restrict__ wgt, T damping) {
    using C = cplx<T>;
    constexpr int S = frame_stride(M);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    C* tw = buf + M * S;
    build_twiddles<T>(tw, M);
    const T inv = T(1) / (T(M) * T(M));
    for (int k = 0; k < N; ++k) {
        const int2 p = pos[k];
        __syncthreads();
        for (int idx = threadIdx.x; idx < M * M; idx += NT) {
            const int r = idx / M, c = idx % M;
            C v = mk<T>(T(0), T(0));
            if (r < w && c < w) {
                const C zz = __ldcg(z + (size_t)(p.x + r) * n + (p.y + c));
                v = probe ? cmul(probe[idx], zz) : zz;
            }
            buf[r * S + c] = v;
        }
        __syncthreads();
        fft2d_smem<T, M, NT, false>(buf, S, tw);
        const T* A = amp + (size_t)k * M * M;
        for (int idx = threadIdx.x; idx < M * M; idx += NT) {
            const C W = buf[(idx / M) * S + idx % M];
            const T a = A[idx];
            const T mag = sqrt(W.x * W.x + W.y * W.y);
            buf[(idx / M) * S + idx % M] = mag > T(0) ? cscale(W, a / mag) : mk<T>(a, T(0));
        }
        __syncthreads();
        fft2d_smem<T, M, NT, true>(buf, S, tw);
        for (int idx = threadIdx.x; idx < w * w; idx += NT) {
            const int r = idx / w, c = idx % w;
            C* zp = z + (size_t)(p.x + r) * n + (p.y + c);
            const C zz = __ldcg(zp);
            const C psi = probe ? cmul(probe[r * M + c], zz) : zz;
            const C dl = csub(cscale(buf[r * S + c], inv), psi);
            C upd;
            if (wgt) upd = cmul(wgt[idx], dl);
            else upd = cscale(dl, damping);
            __stcg(zp, cadd(zz, upd));
        }
    }
}

template <int M>
constexpr int pie_threads() {
    return M <= 8 ? 32 : M == 16 ? 64 : M == 32 ? 128 : M == 64 ? 512 : 1024;
}

template <typename T, int M>
void launch_pie_t(Plan& p, void* z, const void* wgt, double damping) {
    constexpr int NT = pie_threads<M>();
    const size_t smem = sizeof(cplx<T>) * ((size_t)M * frame_stride(M) + M);
    auto kern = k_pie_sweep<T, M, NT>;
    set_smem_attr(kern, smem);
    kern<<<1, NT, smem, p.stream>>>(static_cast<cplx<T>*>(z),
                                    p.has_probe ? p.probe.as<const cplx<T>>() : nullptr,
                                    p.pos.as<const int2>(), p.amp.as<const T>(), p.N, p.n, p.w,
                                    static_cast<const cplx<T>*>(wgt), (T)damping);
    PTG_CHECK_LAUNCH();
    ++p.launches;
}

template <int M>
void launch_pie_reg(Plan& p, void* z, const void* wgt, double damping) {
    constexpr size_t smem = pie_reg_smem_bytes<M>();
    set_smem_attr(k_pie_reg<M>, smem);
    k_pie_reg<M><<<1, M, smem, p.stream>>>(static_cast<float2*>(z), p.has_probe ? p.probe.as<const float2>() : nullptr,
                                          p.pos.as<const int2>(), p.amp.as<const float>(), p.N, p.n,
                                          static_cast<const float2*>(wgt), (float)damping);
    PTG_CHECK_LAUNCH();
    ++p.launches;
}

template <typename T>
void launch_pie(Plan& p, void* z, const void* wgt, double damping) {
    static const bool generic = getenv("PTG_PIE_GENERIC") && getenv("PTG_PIE_GENERIC")[0] == '1';   // A/B switch
    if constexpr (sizeof(T) == 4) {
        if (!generic && p.w == p.M && (p.M == 16 || p.M == 32 || p.M == 64)) {
            if (p.M == 16) launch_pie_reg<16>(p, z, wgt, damping);
            else if (p.M == 32) launch_pie_reg<32>(p, z, wgt, damping);
            else launch_pie_reg<64>(p, z, wgt, damping);
            return;
        }
    }
    switch (p.M) {
        case 1: launch_pie_t<T, 1>(p, z, wgt, damping); break;
        case 2: launch_pie_t<T, 2>(p, z, wgt, damping); break;
        case 4: launch_pie_t<T, 4>(p, z, wgt, damping); break;
        case 8: launch_pie_t<T, 8>(p, z, wgt, damping); break;
        case 16: launch_pie_t<T, 16>(p, z, wgt, damping); break;
        case 32: launch_pie_t<T, 32>(p, z, wgt, damping); break;
        case 64: launch_pie_t<T, 64>(p, z, wgt, damping); break;
        case 128:
            if constexpr (sizeof(T) == 4) {
                launch_pie_t<T, 128>(p, z, wgt, damping);
                break;
            }
            [[fallthrough]];
        default:
            raise(PTG_ERR_CONFIG, "pie: frame side M=" + std::to_string(p.M) +
                                      " exceeds the single-CTA shared-memory path for this precision");
    }
}

// ----------------------------------------------------------- colour planes
// Greedy colouring of the window-overlap graph in scan order (windows j, k
// overlap iff |dr| < w and |dc| < w); a raster with stride s gets
// ceil(w/s)^2 colours.  Deterministic for given positions.
int colour_positions(const Plan& p, std::vector<int>& color) {
    const int w = p.w, G = std::max(1, (p.n + w - 1) / w);
    std::vector<std::vector<int>> cells((size_t)G * G);
    color.assign(p.N, 0);
    int ncol = 0;
    std::vector<char> used;
    for (int j = 0; j < p.N; ++j) {
        const int r = p.pos_h[2 * j], c = p.pos_h[2 * j + 1];
        const int cy = std::min(r / w, G - 1), cx = std::min(c / w, G - 1);
        used.assign(ncol + 1, 0);
        for (int yy = std::max(0, cy - 1); yy <= std::min(G - 1, cy + 1); ++yy)
            for (int xx = std::max(0, cx - 1); xx <= std::min(G - 1, cx + 1); ++xx)
                for (int k : cells[(size_t)yy * G + xx])
                    if (std::abs(p.pos_h[2 * k] - r) < w && std::abs(p.pos_h[2 * k + 1] - c) < w) used[color[k]] = 1;
        int col = 0;
        while (used[col]) ++col;
        color[j] = col;
        ncol = std::max(ncol, col + 1);
        cells[(size_t)cy * G + cx].push_back(j);
    }
    return ncol;
}

// Planes when they stream no more than ~2x the stash's bytes and stay small:
// a plain streaming reduction beats the list-driven gather by far.
bool choose_planes(Plan& p) {
    if (p.N == 0 || p.mp) return false;
    const bool off = getenv("PTG_NO_PLANES") && getenv("PTG_NO_PLANES")[0] == '1';   // A/B switch (read per plan)
    if (off) return false;
    std::vector<int> color;
    const int ncol = colour_positions(p, color);
    const double plane_elems = (double)ncol * p.nn();
    const double stash_elems = (double)p.N * p.w * stash_pitch(p.w);
    if (plane_elems > 2.0 * stash_elems || plane_elems * p.celem() > (double)(512u << 20)) return false;
    p.ncolors = ncol;
    p.color_h = color;
    p.color.alloc(color.size() * sizeof(int));
    PTG_CUDA(cudaMemcpyAsync(p.color.p, color.data(), color.size() * sizeof(int), cudaMemcpyHostToDevice, p.stream));
    p.planes.alloc((size_t)ncol * p.nn() * p.celem());
    // on the plan's (non-blocking) stream: a legacy-stream memset is not ordered
    // before the frame kernels that store into the planes
    PTG_CUDA(cudaMemsetAsync(p.planes.p, 0, p.planes.bytes, p.stream));   // untouched pixels stay zero forever
    return true;
}

// ------------------------------------------------------- RMW order + deps
// Summation / dispatch order of the RMW overlap-add (frame_rmw.cuh): positions
// sorted by window row (stable: scan order within a row), cut into groups of
// nearby rows (a new group once the row moved by >= w/8), each group greedily
// coloured into pairwise non-overlapping classes and emitted class by class.
// deps(k) = every earlier (in this order) frame whose window overlaps k's.
// Deterministic for given positions.
void build_rmw(Plan& p) {
    const int N = p.N, w = p.w;
    auto r0 = [&](int j) { return p.pos_h[2 * (size_t)j]; };
    auto c0 = [&](int j) { return p.pos_h[2 * (size_t)j + 1]; };
    auto overlap = [&](int a_, int b_) { return std::abs(r0(a_) - r0(b_)) < w && std::abs(c0(a_) - c0(b_)) < w; };
    std::vector<int> idx(N);
    for (int j = 0; j < N; ++j) idx[j] = j;
    std::stable_sort(idx.begin(), idx.end(), [&](int a_, int b_) { return r0(a_) < r0(b_); });
    std::vector<int> order;
    order.reserve(N);
    p.rmw_group_end.clear();
    p.rmw_group_maxr0.clear();
    // groups: window rows within PTG_RMW_SB (default w / 8: one scan row of a
    // raster).  Measured on config 5 (ms per evaluation): w/8 24.5, 2 w 25.6,
    // 4 w 26.9, 6 w 27.0 -- larger colour classes give the dependency waits
    // more slack but scatter consecutive frames over more object rows (z and
    // gradient locality in L2), which costs more than the waits
    const char* esb = getenv("PTG_RMW_SB");
    const int gap = std::max(1, esb ? atoi(esb) : p.M == 128 ? 2 * w : w / 8);
    // row groups [s, e) of the row-sorted positions
    std::vector<std::pair<int, int>> rows_g;
    for (int s = 0; s < N;) {
        int e = s + 1;
        while (e < N && r0(idx[e]) - r0(idx[s]) < gap) ++e;
        rows_g.emplace_back(s, e);
        s = e;
    }
    // PTG_RMW_PAIR=S (A/B): colour scan rows R and R + S together (rows S
    // apart do not overlap when S w-steps >= w), doubling the frames per
    // colour class while keeping the rows of a block of 2 S scan rows in L2
    std::vector<std::vector<std::pair<int, int>>> groups;
    const char* epair = getenv("PTG_RMW_PAIR");
    const int S = epair ? atoi(epair) : 0;
    if (S > 0) {
        const int G0 = (int)rows_g.size();
        for (int b = 0; b < G0; b += 2 * S)
            for (int i = 0; i < S && b + i < G0; ++i) {
                groups.push_back({rows_g[b + i]});
                if (b + i + S < G0) groups.back().push_back(rows_g[b + i + S]);
            }
    } else {
        for (auto& g : rows_g) groups.push_back({g});
    }
    for (const auto& grp : groups) {
        std::vector<int> mem;   // positions into idx, ascending row
        for (const auto& [s, e] : grp)
            for (int i = s; i < e; ++i) mem.push_back(i);
        // greedy colouring of the group through a grid of w x w cells
        std::vector<int> col(mem.size(), 0);
        int ncol = 0;
        {
            const int Gc = std::max(1, (p.n + w - 1) / w);
            const int rbase = r0(idx[mem.front()]) / w;
            const int Gr = (r0(idx[mem.back()]) / w) - rbase + 1;
            std::vector<std::vector<int>> cell((size_t)Gr * Gc);   // member slots
            for (size_t a2 = 0; a2 < mem.size(); ++a2) {
                const int i = mem[a2];
                const int cy = r0(idx[i]) / w - rbase, cx = std::min(c0(idx[i]) / w, Gc - 1);
                std::vector<char> used(ncol + 1, 0);
                for (int yy = std::max(0, cy - 1); yy <= std::min(Gr - 1, cy + 1); ++yy)
                    for (int xx = std::max(0, cx - 1); xx <= std::min(Gc - 1, cx + 1); ++xx)
                        for (int b2 : cell[(size_t)yy * Gc + xx])
                            if (overlap(idx[i], idx[mem[b2]])) used[col[b2]] = 1;
                int c = 0;
                while (c < (int)used.size() && used[c]) ++c;
                col[a2] = c;
                ncol = std::max(ncol, c + 1);
                cell[(size_t)cy * Gc + cx].push_back((int)a2);
            }
        }
        int maxr = 0;
        for (int c = 0; c < ncol; ++c)
            for (size_t a2 = 0; a2 < mem.size(); ++a2)
                if (col[a2] == c) order.push_back(idx[mem[a2]]);
        for (int i : mem) maxr = std::max(maxr, r0(idx[i]));
        p.rmw_group_end.push_back((int)order.size());
        p.rmw_group_maxr0.push_back(maxr);
    }
    p.rmw_sufmin_r0.assign(N + 1, p.n);
    for (int k = N - 1; k >= 0; --k) p.rmw_sufmin_r0[k] = std::min(p.rmw_sufmin_r0[k + 1], r0(order[k]));
    // dependencies through a grid of w x w cells
    const int G = std::max(1, (p.n + w - 1) / w);
    std::vector<std::vector<int>> cells((size_t)G * G);   // order indices
    std::vector<int> off(N + 1, 0), dep;
    dep.reserve((size_t)N * 32);
    for (int k = 0; k < N; ++k) {
        const int j = order[k];
        const int cy = std::min(r0(j) / w, G - 1), cx = std::min(c0(j) / w, G - 1);
        for (int yy = std::max(0, cy - 1); yy <= std::min(G - 1, cy + 1); ++yy)
            for (int xx = std::max(0, cx - 1); xx <= std::min(G - 1, cx + 1); ++xx)
                for (int k2 : cells[(size_t)yy * G + xx])
                    if (overlap(j, order[k2])) dep.push_back(k2);
        std::sort(dep.begin() + off[k], dep.end());
        off[k + 1] = (int)dep.size();
        cells[(size_t)cy * G + cx].push_back(k);
    }
    // transitive pruning: d is implied by a later dependency d' of k that
    // itself depends on d (d' completes only after d did) -- a raster frame
    // keeps a handful of its ~60 overlapping predecessors, so a frame polls a
    // few completion counters (each acquire invalidates the SM's L1) instead
    // of all of them
    std::vector<int> poff(N + 1, 0), pdep;
    pdep.reserve(dep.size() / 4 + 16);
    for (int k = 0; k < N; ++k) {
        const int* b = dep.data() + off[k];
        const int* e = dep.data() + off[k + 1];
        for (const int* it = b; it != e; ++it) {
            bool implied = false;
            for (const int* jt = it + 1; jt != e && !implied; ++jt)
                implied = std::binary_search(dep.data() + off[*jt], dep.data() + off[*jt + 1], *it);
            if (!implied) pdep.push_back(*it);
        }
        poff[k + 1] = (int)pdep.size();
    }
    off.swap(poff);
    dep.swap(pdep);
    p.rmw_order_h = order;
    p.rmw_order.alloc(std::max<size_t>(1, (size_t)N) * sizeof(int));
    p.rmw_dep_off.alloc((size_t)(N + 1) * sizeof(int));
    p.rmw_dep_idx.alloc(std::max<size_t>(1, dep.size()) * sizeof(int));
    p.rmw_done.alloc(std::max<size_t>(1, (size_t)N) * sizeof(unsigned));
    p.rmw_work.alloc(sizeof(unsigned));
    if (N) PTG_CUDA(cudaMemcpyAsync(p.rmw_order.p, order.data(), (size_t)N * sizeof(int), cudaMemcpyHostToDevice, p.stream));
    PTG_CUDA(cudaMemcpyAsync(p.rmw_dep_off.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice, p.stream));
    if (!dep.empty())
        PTG_CUDA(cudaMemcpyAsync(p.rmw_dep_idx.p, dep.data(), dep.size() * sizeof(int), cudaMemcpyHostToDevice, p.stream));
    // the host vectors die with this scope: the copies must have been made
    PTG_CUDA(cudaStreamSynchronize(p.stream));
}

// whole-frame scratch of the multi-pass kernels (simulate / project / c128
// objective at large M): ~64 MiB, stays L2-resident between passes
void build_mp_scratch(Plan& p) {
    if (!p.mp) return;
    const size_t fb = p.MM() * p.celem();
    p.mp_chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(p.N, 1), ((size_t)64 << 20) / fb));
    p.mp_scratch.alloc((size_t)p.mp_chunk * fb);
}

// --------------------------------------------------------- chunks / tiles
void build_chunks(Plan& p) {
    p.tiles_x = (p.n + kTileW - 1) / kTileW;
    p.tiles_y = (p.n + kTileH - 1) / kTileH;
    p.mp = !frame_single_cta(p.prec, p.M);
    p.cl = cl_path_ok(p);
    if (p.rows != p.n && !(p.cl && p.w == p.M))
        raise(PTG_ERR_CONFIG, "object bands (sharded plans) need the complex64 cluster path: M = 128 / 256, w = M");
    p.planes_mode = p.rows == p.n && choose_planes(p);
    // RMW overlap-add for the cluster path when the planes do not fit
    // (PTG_NO_RMW=1 selects the stash + gather path instead; read per plan)
    const bool no_rmw = getenv("PTG_NO_RMW") && getenv("PTG_NO_RMW")[0] == '1';
    bool budget_override_off = false;
    // (the RMW order needs many more frames per colour class than clusters in
    // flight: M = 256 scans of >= 2000 positions (configs 4-5: config 4 3.15
    // vs 3.06 ms on the device but 6.5 vs 12.9 ms end to end and a quarter of
    // the DRAM traffic; config 5 22.3 vs 23.0 ms); small scans keep stash +
    // gather (config 3: 0.16 vs 1.06 ms).  PTG_RMW=1 / 0 forces.)
    const char* erm = getenv("PTG_RMW");
    const bool force_rmw = erm && erm[0] == '1';
    if (erm && erm[0] == '0') budget_override_off = true;
    const size_t stash_bytes = (size_t)p.N * p.w * stash_pitch(p.w) * p.celem();
    size_t budget_b = (size_t)2 << 30;
    if (const char* e = getenv("PTG_STASH_BUDGET_MB")) budget_b = std::max<size_t>(1, (size_t)atoll(e)) << 20;
    // (M = 128 keeps the stash even across chunks: config 5's level 1,
    // 27,556 x 128^2, 4.38 ms stash vs 5.04 ms RMW)
    // PTG_RMW128=1 (A/B): M = 128 scans of >= 2000 positions by the RMW kernel too, with colour
    // groups of two window heights (frames in flight: 148 clusters against 33 for M = 256)
    const char* e128 = getenv("PTG_RMW128");
    const bool rmw128 = e128 && e128[0] == '1';
    const bool big = (p.M == 256 && (stash_bytes > budget_b || p.N >= 2000)) || (rmw128 && p.M == 128 && p.N >= 2000);
    p.rmw_mode = (!p.planes_mode && p.cl && p.w == p.M && p.N > 0 && !no_rmw && !budget_override_off &&
                  (force_rmw || big)) ||
                 (p.rows != p.n && p.N > 0);
    if (p.rmw_mode) {   // one chunk, no tile lists, no stash
        auto c = std::make_unique<Chunk>();
        c->first = 0;
        c->count = p.N;
        p.chunk_size = p.N;
        p.chunks.clear();
        p.chunks.push_back(std::move(c));
        p.stash.alloc(p.celem());
        p.misfit_per_pos = cl_mpp(p.M / rmw_line(p), p.M);
        p.misfit.alloc((size_t)p.N * p.misfit_per_pos * sizeof(double));
        p.dotp.alloc((size_t)kRmwInitBlocks * sizeof(double));
        build_mp_scratch(p);
        build_rmw(p);
        return;
    }
    if (p.planes_mode) {   // one chunk, no tile lists, no stash
        auto c = std::make_unique<Chunk>();
        c->first = 0;
        c->count = p.N;
        p.chunk_size = p.N;
        p.chunks.clear();
        p.chunks.push_back(std::move(c));
        p.stash.alloc(p.celem());
        p.misfit_per_pos = p.cl ? p.M / 32 : 1;
        p.misfit.alloc(std::max<size_t>(1, (size_t)p.N * p.misfit_per_pos) * sizeof(double));
        p.dotp.alloc((size_t)kPlaneBlocks * sizeof(double));
        return;
    }
    const size_t per = (size_t)p.w * stash_pitch(p.w) * p.celem();
    // stash bytes per chunk: 2 GiB; PTG_STASH_BUDGET_MB lowers it (read per
    // plan) so tests can drive the multi-chunk path with small problems
    size_t budget = (size_t)2 << 30;
    if (const char* e = getenv("PTG_STASH_BUDGET_MB")) budget = std::max<size_t>(1, (size_t)atoll(e)) << 20;
    int cs = p.N > 0 ? (int)std::min<size_t>((size_t)p.N, std::max<size_t>(1, budget / per)) : 1;
    p.chunk_size = cs;
    p.chunks.clear();
    const int ntiles = p.tiles_x * p.tiles_y;
    const int nchunks = p.N > 0 ? (p.N + cs - 1) / cs : 1;
    for (int ci = 0; ci < nchunks; ++ci) {
        auto c = std::make_unique<Chunk>();
        c->first = ci * cs;
        c->count = std::min(cs, p.N - c->first);
        if (c->count < 0) c->count = 0;
        std::vector<std::vector<int>> lists(ntiles);
        for (int j = c->first; j < c->first + c->count; ++j) {
            const int r0 = p.pos_h[2 * j], c0 = p.pos_h[2 * j + 1];
            const int ty0 = r0 / kTileH, ty1 = (r0 + p.w - 1) / kTileH;
            // pixel pairs (even x) touching [c0, c0 + w): x in [c0 - (c0 & 1), c0 + w)
            const int tx0 = (c0 - (c0 & 1)) / kTileW, tx1 = (c0 + p.w - 1) / kTileW;
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) lists[ty * p.tiles_x + tx].push_back(j);
        }
        std::vector<int> ids;
        // Per visited tile, a fixed-stride (cap) list of the windows covering it in
        // ascending scan order: {stash offset of window origin - r0*w - c0, r0, c0, j},
        // padded with entries that never match (so no per-tile count is needed).
        c->all_tiles = (nchunks == 1);
        size_t cap = 1;
        for (int t = 0; t < ntiles; ++t) {
            if (!c->all_tiles && lists[t].empty()) continue;
            ids.push_back(t);
            cap = std::max(cap, lists[t].size());
        }
        cap = (cap + 15) / 16 * 16;   // multiple of the gather's batch U
        const int4 pad = make_int4(0, -(1 << 29), -(1 << 29), -1);
        std::vector<int4> list(ids.size() * cap, pad);
        for (size_t b = 0; b < ids.size(); ++b) {
            size_t e = 0;
            for (int j : lists[ids[b]]) {
                const int r0 = p.pos_h[2 * j], c0 = p.pos_h[2 * j + 1];
                const int sp = stash_pitch(p.w), c0e = c0 - (c0 & 1);
                const long long off = (long long)(j - c->first) * p.w * sp - (long long)r0 * sp - c0e;
                list[b * cap + e++] = make_int4((int)off, r0, c0e, j);
            }
        }
        c->cap = (int)cap;
        c->ntiles = (int)ids.size();
        if (!c->all_tiles) {
            c->tile_ids.alloc(ids.size() * sizeof(int));
            if (!ids.empty()) PTG_CUDA(cudaMemcpyAsync(c->tile_ids.p, ids.data(), ids.size() * sizeof(int), cudaMemcpyHostToDevice, p.stream));
        }
        // int32 stash offsets: the per-chunk stash budget keeps them < 2^31 elements
        c->tile_list.alloc(std::max<size_t>(1, list.size()) * sizeof(int4));
        if (!list.empty()) PTG_CUDA(cudaMemcpyAsync(c->tile_list.p, list.data(), list.size() * sizeof(int4), cudaMemcpyHostToDevice, p.stream));
        p.chunks.push_back(std::move(c));
    }
    p.stash.alloc(std::max<size_t>(1, (size_t)cs * p.w * stash_pitch(p.w)) * p.celem());
    p.misfit_per_pos = p.cl ? p.M / 32 : p.mp ? p.M / kMpLines : 1;
    build_mp_scratch(p);
    p.misfit.alloc(std::max<size_t>(1, (size_t)p.N * p.misfit_per_pos) * sizeof(double));
    // dot partials: one per tile (single chunk) or one per k_shift block
    p.dotp.alloc(std::max<size_t>((size_t)ntiles, 1024) * sizeof(double));
}

void check_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        raise(PTG_ERR_CUDA, std::string("no CUDA device available (libptg has no CPU fallback): ") +
                                cudaGetErrorString(e));
    if (device < 0 || device >= count) raise(PTG_ERR_CUDA, "device ordinal out of range");
    cudaDeviceProp prop;
    PTG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        raise(PTG_ERR_CUDA, "libptg is built for sm_100a (B200); device " + std::to_string(device) +
                                " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
    PTG_CUDA(cudaSetDevice(device));
}

}  // namespace

void check_device_public(int device) { check_device(device); }

// ------------------------------------------------------------------ create
// The solvers' work vectors are stream-ordered allocations (cudaMallocAsync).
// With the default pool release threshold (0) every synchronisation hands the
// freed memory back to the driver and the next allocation maps it again
// (~100 us for a few MB): an MG/OPT cycle allocates ~30 vectors per level.
// Keep the pool's memory reserved instead (bounded by the peak working set).
static void keep_pool_memory(int device) {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    uint64_t thr = ~0ull;
    PTG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done[device] = true;
}

static std::unique_ptr<Plan> plan_create_rows(const ptg_plan_desc& d, int rows, const Shard& shard);

std::unique_ptr<Plan> plan_create(const ptg_plan_desc& d) { return plan_create_rows(d, d.n, Shard{}); }

static std::unique_ptr<Plan> plan_create_rows(const ptg_plan_desc& d, int rows, const Shard& shard) {
    if (d.n < 1) raise(PTG_ERR_GEOMETRY, "object side must be positive");
    if (rows < 1 || rows > d.n) raise(PTG_ERR_GEOMETRY, "object band rows must be in [1, n]");
    if (!is_pow2(d.M))
        raise(PTG_ERR_GEOMETRY, "fft2: grid side must be a positive power of two, got " + std::to_string(d.M));
    if (d.w < 1 || d.w > d.M || d.w > d.n)
        raise(PTG_ERR_GEOMETRY, "window side " + std::to_string(d.w) + " must satisfy 1 <= w <= min(M, n)");
    if (d.N < 0) raise(PTG_ERR_DOMAIN, "negative pattern count");
    if (d.precision != PTG_C64 && d.precision != PTG_C128) raise(PTG_ERR_CONFIG, "unknown precision");
    if (d.N > 0 && !d.positions) raise(PTG_ERR_CONFIG, "positions pointer is NULL");
    for (int k = 0; k < d.N; ++k) {
        const int r = d.positions[2 * k], c = d.positions[2 * k + 1];
        if (r < 0 || c < 0 || r + d.w > rows || c + d.w > d.n)
            raise(PTG_ERR_GEOMETRY, "probe window [" + std::to_string(r) + "," + std::to_string(c) +
                                        ")+" + std::to_string(d.w) + " does not fit an n=" +
                                        std::to_string(d.n) + " grid");
    }
    if (!frame_supported(d.precision, d.M))
        raise(PTG_ERR_CONFIG, "frame side M=" + std::to_string(d.M) + " is not supported for this precision yet");
    check_device(d.device);

    auto p = std::make_unique<Plan>();
    p->n = d.n;
    p->rows = rows;
    p->shard = shard;
    p->M = d.M;
    p->w = d.w;
    p->N = d.N;
    p->prec = d.precision;
    p->device = d.device;
    p->has_probe = d.probe != nullptr;
    p->pos_h.assign(d.positions, d.positions + 2 * (size_t)d.N);
    PTG_CUDA(cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking));
    p->stream = p->own_stream;
    keep_pool_memory(p->device);
    LaunchScope ls(*p);

    p->pos.alloc(std::max<size_t>(1, (size_t)d.N) * sizeof(int2));
    if (d.N) PTG_CUDA(cudaMemcpyAsync(p->pos.p, d.positions, (size_t)d.N * sizeof(int2), cudaMemcpyHostToDevice, p->stream));
    if (p->has_probe) {
        p->probe_h.assign(d.probe, d.probe + 2 * p->MM());
        p->probe.alloc(p->MM() * p->celem());
        p->stage.ensure(p->MM() * 16);
        PTG_CUDA(cudaMemcpyAsync(p->stage.p, d.probe, p->MM() * 16, cudaMemcpyHostToDevice, p->stream));
        dev_from_c128(p->prec, p->probe.p, p->stage.as<double>(), p->MM(), p->stream);
    }
    build_chunks(*p);
    p->value.alloc(4 * sizeof(double));
    p->counter.alloc(sizeof(unsigned int) * 4);
    PTG_CUDA(cudaMemsetAsync(p->counter.p, 0, p->counter.bytes, p->stream));
    p->scratch.alloc((kReduceBlocks + 2) * sizeof(double));
    PTG_CUDA(cudaMemsetAsync(p->scratch.p, 0, p->scratch.bytes, p->stream));
    p->flag.alloc(sizeof(unsigned long long));
    // fixed size for the plan's lifetime: replayed host-eval graphs copy the value
    // into this buffer, so it must never be reallocated (solvers use <= 8 doubles)
    p->hval.ensure(kHvalDoubles * sizeof(double));
    if (d.data) plan_set_data_host(*p, d.data, d.data_dtype);
    PTG_CUDA(cudaStreamSynchronize(p->stream));
    return p;
}

// ------------------------------------------------------------------- data
void plan_refresh_amp(Plan& p) {
    const size_t len = (size_t)p.N * p.MM();
    p.amp.ensure(std::max<size_t>(1, len) * p.relem());
    unsigned long long init = ~0ull;
    PTG_CUDA(cudaMemcpyAsync(p.flag.p, &init, sizeof init, cudaMemcpyHostToDevice, p.stream));
    if (len) {
        if (p.prec == PTG_C64)
            k_prepare<float><<<grid_for(len), 256, 0, p.stream>>>(p.inten.as<const float>(), len, p.amp.as<float>(), p.flag.as<unsigned long long>());
        else
            k_prepare<double><<<grid_for(len), 256, 0, p.stream>>>(p.inten.as<const double>(), len, p.amp.as<double>(), p.flag.as<unsigned long long>());
        PTG_CHECK_LAUNCH();
        ++p.launches;
    }
    unsigned long long bad = 0;
    PTG_CUDA(cudaMemcpyAsync(&bad, p.flag.p, sizeof bad, cudaMemcpyDeviceToHost, p.stream));
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    if (bad != ~0ull) {
        p.amp_valid = p.inten_valid = false;
        raise(PTG_ERR_DOMAIN, "diffraction pattern has a negative intensity at index " +
                                  std::to_string(bad % p.MM()));
    }
    p.amp_valid = true;
    p.inten_valid = true;
    ++p.data_gen;
}

void plan_set_data_device(Plan& p, const void* data, int dtype) {
    LaunchScope ls(p);
    const size_t len = (size_t)p.N * p.MM();
    p.inten.ensure(std::max<size_t>(1, len) * p.relem());
    if (len) dev_real_convert(p.prec, p.inten.p, dtype, data, len, p.stream);
    plan_refresh_amp(p);
}

// PTYF stack (image_io.hpp:10-20: "PTYF", u32 n, u32 channels, u32 0, then
// channel-major row-major float64) streamed to the device through two pinned
// staging buffers: the file read of chunk i+1 overlaps the H2D copy and the
// on-device f64 -> plan-precision conversion of chunk i (image_io.cpp:184-196).
void plan_load_ptyf(Plan& p, const char* path) {
    LaunchScope ls(p);
    const std::string where = std::string(path ? path : "(null)") + ": ";
    FILE* f = path ? std::fopen(path, "rb") : nullptr;
    if (!f) raise(PTG_ERR_IO, where + "cannot open for reading");
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    unsigned char hdr[16];
    if (std::fread(hdr, 1, 4, f) != 4 || std::memcmp(hdr, "PTYF", 4) != 0) raise(PTG_ERR_IO, where + "not a PTYF file");
    if (std::fread(hdr + 4, 1, 12, f) != 12) raise(PTG_ERR_IO, where + "truncated header");
    auto u32 = [&](int o) { return (uint32_t)hdr[o] | (uint32_t)hdr[o + 1] << 8 | (uint32_t)hdr[o + 2] << 16 | (uint32_t)hdr[o + 3] << 24; };
    const long long n = u32(4), ch = u32(8);
    if (n < 1 || ch < 1) raise(PTG_ERR_IO, where + "bad PTYF dimensions");
    if (n != p.M || ch != p.N)
        raise(PTG_ERR_GEOMETRY, where + "stack of " + std::to_string(ch) + " patterns of side " + std::to_string(n) +
                                    " does not match the plan (" + std::to_string(p.N) + " x " + std::to_string(p.M) + ")");
    const size_t len = (size_t)p.N * p.MM();
    p.inten.ensure(std::max<size_t>(1, len) * p.relem());
    const size_t chunk = std::min<size_t>(len, (size_t)4 << 20);   // doubles per chunk (32 MiB)
    HostPinned hb[2];
    DevMem db[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) {
        hb[b].ensure(chunk * sizeof(double));
        db[b].alloc(chunk * sizeof(double));
        PTG_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    struct EvFree {
        cudaEvent_t* e;
        ~EvFree() { for (int b = 0; b < 2; ++b) if (e[b]) cudaEventDestroy(e[b]); }
    } evfree{ev};
    size_t done = 0;
    for (int i = 0; done < len; ++i) {
        const int b = i & 1;
        const size_t cnt = std::min(chunk, len - done);
        if (i >= 2) PTG_CUDA(cudaEventSynchronize(ev[b]));   // buffer b's previous copy has drained
        if (std::fread(hb[b].p, sizeof(double), cnt, f) != cnt) {
            PTG_CUDA(cudaStreamSynchronize(p.stream));
            p.amp_valid = p.inten_valid = false;
            raise(PTG_ERR_IO, where + "truncated payload");
        }
        PTG_CUDA(cudaMemcpyAsync(db[b].p, hb[b].p, cnt * sizeof(double), cudaMemcpyHostToDevice, p.stream));
        dev_real_convert(p.prec, static_cast<unsigned char*>(p.inten.p) + done * p.relem(), PTG_F64, db[b].p, cnt,
                         p.stream);
        PTG_CUDA(cudaEventRecord(ev[b], p.stream));
        done += cnt;
    }
    plan_refresh_amp(p);   // synchronises the stream
}

void plan_set_data_host(Plan& p, const void* data, int dtype) {
    const size_t len = (size_t)p.N * p.MM();
    if (!len) {
        p.amp_valid = p.inten_valid = true;
        return;
    }
    const size_t sb = len * (dtype == PTG_F32 ? 4 : 8);
    DevMem tmp;
    tmp.alloc(sb);
    PTG_CUDA(cudaMemcpyAsync(tmp.p, data, sb, cudaMemcpyHostToDevice, p.stream));
    plan_set_data_device(p, tmp.p, dtype);
    PTG_CUDA(cudaStreamSynchronize(p.stream));
}

void plan_ensure(Plan& p, int metric) {
    const size_t len = (size_t)p.N * p.MM();
    if (metric == PTG_INTENSITY && !p.inten_valid) {
        if (!p.amp_valid) raise(PTG_ERR_CONFIG, "plan has no diffraction data");
        p.inten.ensure(std::max<size_t>(1, len) * p.relem());
        if (len) {
            if (p.prec == PTG_C64) k_square<float><<<grid_for(len), 256, 0, p.stream>>>(p.amp.as<const float>(), len, p.inten.as<float>());
            else k_square<double><<<grid_for(len), 256, 0, p.stream>>>(p.amp.as<const double>(), len, p.inten.as<double>());
            PTG_CHECK_LAUNCH();
            ++p.launches;
        }
        p.inten_valid = true;
        ++p.data_gen;
    }
    if (metric == PTG_DISTANCE && !p.amp_valid) {
        if (!p.inten_valid) raise(PTG_ERR_CONFIG, "plan has no diffraction data");
        plan_refresh_amp(p);
    }
    if (metric != PTG_DISTANCE && metric != PTG_INTENSITY) raise(PTG_ERR_CONFIG, "unknown metric kind");
}

// ------------------------------------------------------------------- eval
template <typename T>
static void eval_t(Plan& p, int metric, const void* z, const void* v, void* grad, double* value_dev) {
    using C = cplx<T>;
    const T* data = metric == PTG_DISTANCE ? p.amp.as<const T>() : p.inten.as<const T>();
    if constexpr (sizeof(T) == 4) {
        if (p.rmw_mode) {
            // init (grad = -v | 0, <v,z> partials, counters) -> persistent RMW
            // frames -> value; all on the plan's stream
            p.ev_begin(1);
            // a BANDS shard owns its first own_rows rows: the shift and <v,z> there only
            const size_t own = p.shard.layout == PTG_SHARD_BANDS ? (size_t)p.shard.own_rows * p.n : p.nn();
            k_rmw_init<C><<<kRmwInitBlocks, 256, 0, p.stream>>>(static_cast<const C*>(v), static_cast<const C*>(z),
                                                                static_cast<C*>(grad), p.nn(), own,
                                                                v ? p.dotp.as<double>() : nullptr,
                                                                p.rmw_done.as<unsigned>(), p.N, p.rmw_work.as<unsigned>());
            PTG_CHECK_LAUNCH();
            p.ev_end();
            ++p.launches;
            FrameArgs<T> a = frame_args<T>(p, z, data);
            p.ev_begin(0);
            if (metric == PTG_DISTANCE) launch_rmw<OP_DISTANCE>(p, a, data, static_cast<float2*>(grad), 0, p.N);
            else launch_rmw<OP_INTENSITY>(p, a, data, static_cast<float2*>(grad), 0, p.N);
            p.ev_end();
            ++p.launches;
            k_finalize<<<1, 256, 0, p.stream>>>(p.misfit.as<const double>(), p.N * p.misfit_per_pos,
                                                p.dotp.as<const double>(), v ? kRmwInitBlocks : 0, value_dev);
            PTG_CHECK_LAUNCH();
            ++p.launches;
            return;
        }
    }
    const bool single = p.chunks.size() == 1;
    // fused last-block finalize in the gather (single-chunk plans); PTG_NOFUSE=1
    // selects the separate finalize kernel (kept for A/B measurement)
    static const bool nofuse = getenv("PTG_NOFUSE") && getenv("PTG_NOFUSE")[0] == '1';
    const bool fuse = single && p.chunks[0]->ntiles > 0 && !nofuse;
    if (!single) dev_fill_zero(p.prec, grad, p.nn(), p.stream);
    for (auto& cp : p.chunks) {
        Chunk& c = *cp;
        if (c.count > 0) {
            FrameArgs<T> a = frame_args<T>(p, z, data);
            a.first = c.first;
            // frame_kernel writes stash[j*w*w]; offset the base so j - first maps to 0
            a.stash = reinterpret_cast<C*>(p.stash.as<C>()) - (size_t)c.first * p.w * stash_pitch(p.w);
            p.ev_begin(0);
            if (p.mp && !p.cl) {
                if (metric == PTG_DISTANCE) launch_mp<T, OP_DISTANCE>(p, a, c.first, c.count);
                else launch_mp<T, OP_INTENSITY>(p, a, c.first, c.count);
            } else {
                if (metric == PTG_DISTANCE) launch_objective<T, OP_DISTANCE>(p, a, c.count, z, data);
                else launch_objective<T, OP_INTENSITY>(p, a, c.count, z, data);
                ++p.launches;
            }
            p.ev_end();
        }
        if (p.planes_mode) {
            // streaming colour-plane reduction + shift + <v,z> + final value,
            // chained to the frame kernel by programmatic dependent launch
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(kPlaneBlocks);
            cfg.blockDim = dim3(256);
            cfg.stream = p.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = p.timing ? 0 : 1;
            p.ev_begin(1);
            PTG_CUDA(cudaLaunchKernelEx(&cfg, plane_reduce_kernel<T>(plane_qs(p)), p.planes.as<const C>(), p.ncolors, p.nn(),
                                        static_cast<const C*>(v), static_cast<const C*>(z), static_cast<C*>(grad),
                                        p.dotp.as<double>(), p.misfit.as<const double>(), p.N * p.misfit_per_pos,
                                        value_dev, p.counter.as<unsigned int>(), 0));
            p.ev_end();
            ++p.launches;
            return;
        }
        if (c.ntiles > 0) {
            // single-chunk plans fuse the shift, <v,z> and the final value reduction
            // into the gather (last-block-done); it is chained to the frame kernel
            // by programmatic dependent launch so its launch overlaps the frame tail
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(c.ntiles);
            cfg.blockDim = dim3(kTileW / 2, kTileH);
            cfg.stream = p.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = p.timing ? 0 : 1;   // event timing needs plain kernel boundaries
            static const int reps = getenv("PTG_GATHER_REPS") ? atoi(getenv("PTG_GATHER_REPS")) : 1;   // A/B probe
            for (int rep = 0; rep < reps; ++rep) {
            p.ev_begin(rep == 0 ? 1 : 2);
            PTG_CUDA(cudaLaunchKernelEx(
                &cfg, k_overlap_gather<T>, p.stash.as<const C>(),
                c.all_tiles ? (const int*)nullptr : c.tile_ids.as<const int>(), c.cap,
                c.tile_list.as<const int4>(), p.n, p.w, p.tiles_x,
                single ? static_cast<const C*>(v) : (const C*)nullptr, static_cast<const C*>(z),
                static_cast<C*>(grad), p.dotp.as<double>(), single ? 0 : 1, p.misfit.as<const double>(),
                p.N * p.misfit_per_pos, fuse ? value_dev : (double*)nullptr, p.counter.as<unsigned int>()));
            p.ev_end();
            ++p.launches;
            }
        }
    }
    if (fuse) return;   // value produced by the fused gather
    int ndot = (single && v) ? p.chunks[0]->ntiles : 0;
    if (!single && v) {
        const int blocks = 1024;
        k_shift<T><<<blocks, 256, 0, p.stream>>>(static_cast<const C*>(v), static_cast<const C*>(z),
                                                 static_cast<C*>(grad), p.nn(), p.dotp.as<double>());
        PTG_CHECK_LAUNCH();
        ++p.launches;
        ndot = blocks;
    }
    k_finalize<<<1, 256, 0, p.stream>>>(p.misfit.as<const double>(), p.N * p.misfit_per_pos,
                                        p.dotp.as<const double>(), ndot, value_dev);
    PTG_CHECK_LAUNCH();
    ++p.launches;
}

void plan_eval(Plan& p, int metric, const void* z, const void* v, void* grad, double* value_dev) {
    LaunchScope ls(p);
    plan_ensure(p, metric);
    if (!grad) {
        p.gbuf.ensure(p.nn() * p.celem());
        grad = p.gbuf.p;
    }
    if (!value_dev) value_dev = p.value.as<double>();
    // REPLICATED shards: local frames without the shift, the sum over ranks,
    // then the shift once (grad -= v, value -= <v,z>, identical on every rank)
    const bool rep = p.comm && p.shard.layout == PTG_SHARD_REPLICATED;
    const void* v_local = rep ? nullptr : v;
    if (p.prec == PTG_C64) eval_t<float>(p, metric, z, v_local, grad, value_dev);
    else eval_t<double>(p, metric, z, v_local, grad, value_dev);
    if (!p.comm) return;
    comm_exchange(p, grad, value_dev);
    if (rep && v) {
        p.dotp.ensure((size_t)kShiftBlocks * sizeof(double));
        if (p.prec == PTG_C64)
            k_shift<float><<<kShiftBlocks, 256, 0, p.stream>>>(static_cast<const float2*>(v), static_cast<const float2*>(z),
                                                               static_cast<float2*>(grad), p.nn(), p.dotp.as<double>());
        else
            k_shift<double><<<kShiftBlocks, 256, 0, p.stream>>>(static_cast<const double2*>(v), static_cast<const double2*>(z),
                                                                static_cast<double2*>(grad), p.nn(), p.dotp.as<double>());
        PTG_CHECK_LAUNCH();
        k_sub_dots<<<1, 256, 0, p.stream>>>(p.dotp.as<const double>(), kShiftBlocks, value_dev);
        PTG_CHECK_LAUNCH();
        p.launches += 2;
    }
}

// ------------------------------------------------------------- sharding
void shard_layout(int n, int w, int N, const int32_t* pos, int world, int rank, int layout, int out[6]) {
    if (world < 1 || rank < 0 || rank >= world) raise(PTG_ERR_CONFIG, "shard: bad rank / world size");
    if (layout != PTG_SHARD_REPLICATED && layout != PTG_SHARD_BANDS) raise(PTG_ERR_CONFIG, "shard: unknown layout");
    // scan rows: a new row once the window row moved by >= w/8 (build_rmw's grouping)
    const int gap = std::max(1, w / 8);
    std::vector<int> row_start;
    for (int i = 0; i < N; ++i)
        if (i == 0 || pos[2 * i] - pos[2 * row_start.back()] >= gap)
            row_start.push_back(i);
    const int G = (int)row_start.size();
    if (G < world) raise(PTG_ERR_CONFIG, "shard: more ranks (" + std::to_string(world) + ") than scan rows (" +
                                             std::to_string(G) + ")");
    // block b: scan rows [cut[b], cut[b+1]) with ~N / world positions each
    std::vector<int> cut(world + 1, G);
    cut[0] = 0;
    for (int b = 1; b < world; ++b) {
        const double target = (double)N * b / world;
        int g = cut[b - 1] + 1;
        while (g < G - (world - b) && row_start[g] < target) ++g;
        cut[b] = g;
    }
    auto first = [&](int b) { return cut[b] < G ? row_start[cut[b]] : N; };
    auto min_row = [&](int b) {
        int m = n;
        for (int i = first(b); i < first(b + 1); ++i) m = std::min(m, (int)pos[2 * i]);
        return m;
    };
    auto max_end = [&](int b) {
        int m = 0;
        for (int i = first(b); i < first(b + 1); ++i) m = std::max(m, (int)pos[2 * i] + w);
        return m;
    };
    std::vector<int> R(world + 1, n);
    R[0] = 0;
    for (int b = 1; b < world; ++b) R[b] = min_row(b);
    for (int b = 0; b + 1 < world; ++b)
        if (max_end(b) - w > R[b + 1])
            raise(PTG_ERR_CONFIG, "shard: scan rows of consecutive ranks interleave (window rows not ordered)");
    out[0] = first(rank);
    out[1] = first(rank + 1);
    if (layout == PTG_SHARD_REPLICATED) {
        out[2] = 0;
        out[3] = n;
        out[4] = n;
        out[5] = 0;
        return;
    }
    auto band_end = [&](int b) { return std::min(n, std::max(R[b + 1], max_end(b))); };
    for (int b = 0; b + 1 < world; ++b)
        if (band_end(b) - R[b + 1] > R[b + 2] - R[b + 1])
            raise(PTG_ERR_CONFIG, "shard: a rank's halo (" + std::to_string(band_end(b) - R[b + 1]) +
                                      " rows) exceeds the next rank's own rows; use fewer ranks");
    out[2] = R[rank];
    out[3] = band_end(rank) - R[rank];
    out[4] = R[rank + 1] - R[rank];
    out[5] = rank > 0 ? band_end(rank - 1) - R[rank] : 0;
}

std::unique_ptr<Plan> plan_create_sharded(const ptg_plan_desc& d, int world, int rank, int layout) {
    if (d.N > 0 && !d.positions) raise(PTG_ERR_CONFIG, "positions pointer is NULL");
    int L[6];
    shard_layout(d.n, d.w, d.N, d.positions, world, rank, layout, L);
    Shard sh;
    sh.layout = layout;
    sh.world = world;
    sh.rank = rank;
    sh.pos_begin = L[0];
    sh.pos_end = L[1];
    sh.row0 = L[2];
    sh.own_rows = L[4];
    sh.halo_prev = L[5];
    std::vector<int32_t> local((size_t)2 * (L[1] - L[0]));
    for (int i = L[0]; i < L[1]; ++i) {
        local[2 * (size_t)(i - L[0])] = d.positions[2 * (size_t)i] - L[2];
        local[2 * (size_t)(i - L[0]) + 1] = d.positions[2 * (size_t)i + 1];
    }
    ptg_plan_desc ld = d;
    ld.N = L[1] - L[0];
    ld.positions = local.data();
    return plan_create_rows(ld, L[3], sh);
}

// ------------------------------------------------------ banded host eval
// ptg_eval with host complex128 buffers.  The object is uploaded in row bands
// on a copy-in stream; as soon as the rows a group of frames reads are on the
// device, that group runs (positions must be ordered by window row, as
// raster / serpentine scans are); plane-reduce blocks run once every frame
// reaching their pixel rows has run (a subset of the same fixed partition, so
// the gradient and the value are bitwise those of plan_eval); finished
// gradient rows go back on a copy-out stream while later bands compute.
// Falls back to upload -> plan_eval -> download when a condition fails.
template <typename T>
static void eval_host_banded(Plan& p, int metric, const double* z, const double* v, double* value, double* grad,
                             bool capture = false) {
    using C = cplx<T>;
    const auto t_beg = std::chrono::steady_clock::now();
    auto t_enq = t_beg;
    const int n = p.n, w = p.w, N = p.N;
    const size_t nn = p.nn(), npairs = (nn + 1) / 2, chunk = (npairs + kPlaneBlocks - 1) / kPlaneBlocks;
    static const int K = getenv("PTG_BANDS") ? std::max(2, std::min(16, atoi(getenv("PTG_BANDS")))) : 4;   // object bands (more: host-bound)
    const int H = (n + K - 1) / K;
    // two copy-in and two copy-out streams, alternating by band: concurrent
    // transfers use two copy engines (a single 4 MiB H2D measured 161 us on
    // some hosts, split over two streams 100 us)
    if (!p.s_in) {
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_in, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_out, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_in2, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_out2, cudaStreamNonBlocking));
    }
    const cudaStream_t sin[2] = {p.s_in, p.s_in2}, sout[2] = {p.s_out, p.s_out2};
    while (p.ev_band.size() < (size_t)(3 * K + 4)) {
        cudaEvent_t e;
        PTG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p.ev_band.push_back(e);
    }
    cudaEvent_t* ev_in = p.ev_band.data();            // [K] band uploaded
    cudaEvent_t* ev_out = p.ev_band.data() + K;       // [K] gradient rows converted
    cudaEvent_t ev_start = p.ev_band[2 * K], ev_val = p.ev_band[2 * K + 1], ev_join = p.ev_band[2 * K + 2],
                ev_join2 = p.ev_band[2 * K + 3];
    const size_t cb = p.celem();
    p.zbuf.ensure(nn * cb);
    p.gbuf.ensure(nn * cb);
    if (v) p.vbuf.ensure(nn * cb);
    p.stage.ensure(nn * 16 * (v ? 2 : 1));
    p.stage_out.ensure(nn * 16);
    double* st_z = p.stage.as<double>();
    double* st_v = st_z + 2 * nn;
    C* zd = p.zbuf.as<C>();
    C* vd = v ? p.vbuf.as<C>() : nullptr;
    C* gd = p.gbuf.as<C>();
    const T* data = metric == PTG_DISTANCE ? p.amp.as<const T>() : p.inten.as<const T>();
    // the copy streams start after work already queued on the plan's stream
    PTG_CUDA(cudaEventRecord(ev_start, p.stream));
    for (int i = 0; i < 2; ++i) {
        PTG_CUDA(cudaStreamWaitEvent(sin[i], ev_start, 0));
        PTG_CUDA(cudaStreamWaitEvent(sout[i], ev_start, 0));
    }
    for (int b = 0; b < K; ++b) {
        const size_t r0 = (size_t)std::min(n, b * H), r1 = (size_t)std::min(n, (b + 1) * H);
        const size_t off = r0 * n, cnt = (r1 - r0) * n;
        if (cnt) {
            PTG_CUDA(cudaMemcpyAsync(st_z + 2 * off, z + 2 * off, cnt * 16, cudaMemcpyHostToDevice, sin[b & 1]));
            if (v) PTG_CUDA(cudaMemcpyAsync(st_v + 2 * off, v + 2 * off, cnt * 16, cudaMemcpyHostToDevice, sin[b & 1]));
        }
        PTG_CUDA(cudaEventRecord(ev_in[b], sin[b & 1]));
    }
    int f_done = 0, k_done = 0;
    size_t rows_out = 0;   // gradient rows already converted for copy-out
    FrameArgs<T> a = frame_args<T>(p, zd, data);
    for (int b = 0; b < K; ++b) {
        const int r1 = std::min(n, (b + 1) * H);
        const size_t off = (size_t)std::min(n, b * H) * n, cnt = (size_t)r1 * n - off;
        PTG_CUDA(cudaStreamWaitEvent(p.stream, ev_in[b], 0));
        if (cnt) {
            dev_from_c128(p.prec, zd + off, st_z + 2 * off, cnt, p.stream);
            if (v) dev_from_c128(p.prec, vd + off, st_v + 2 * off, cnt, p.stream);
        }
        // frames whose windows lie in rows < r1 (all of them after the last band)
        int f_end = f_done;
        while (f_end < N && (b == K - 1 || p.pos_h[2 * f_end] + w <= r1)) ++f_end;
        if (f_end > f_done) {
            a.first = f_done;
            if (metric == PTG_DISTANCE) launch_objective<T, OP_DISTANCE>(p, a, f_end - f_done, zd, data);
            else launch_objective<T, OP_INTENSITY>(p, a, f_end - f_done, zd, data);
            ++p.launches;
            f_done = f_end;
        }
        // reduce blocks whose pixel rows no later frame reaches AND whose z / v
        // rows are already on the device (rows < r1; every row after the last
        // band) -- a scan that leaves uncovered rows must not reduce them early
        const int next_row = f_done < N ? p.pos_h[2 * f_done] : n;   // first row a pending frame touches
        const int ready_row = b == K - 1 ? n : std::min(next_row, r1);
        int k_end = k_done;
        while (k_end < kPlaneBlocks) {
            const size_t hi = std::min(npairs, (size_t)(k_end + 1) * chunk);
            const size_t last_pix = hi ? std::min(nn - 1, 2 * hi - 1) : 0;
            if ((int)(last_pix / n) >= ready_row) break;
            ++k_end;
        }
        if (k_end > k_done) {
            plane_reduce_kernel<T>(plane_qs(p))<<<k_end - k_done, 256, 0, p.stream>>>(
                p.planes.as<const C>(), p.ncolors, nn, vd, zd, gd, p.dotp.as<double>(),
                p.misfit.as<const double>(), N * p.misfit_per_pos, nullptr, p.counter.as<unsigned int>(), k_done);
            PTG_CHECK_LAUNCH();
            ++p.launches;
            k_done = k_end;
        }
        // complete gradient rows -> complex128 staging -> host
        const size_t pairs_done = std::min(npairs, (size_t)k_done * chunk);
        const size_t rows_ready = k_done == kPlaneBlocks ? (size_t)n : (2 * pairs_done) / n;
        if (rows_ready > rows_out) {
            const size_t o = rows_out * n, c = (rows_ready - rows_out) * n;
            dev_to_c128(p.prec, p.stage_out.as<double>() + 2 * o, gd + o, c, p.stream);
            PTG_CUDA(cudaEventRecord(ev_out[b], p.stream));
            PTG_CUDA(cudaStreamWaitEvent(sout[b & 1], ev_out[b], 0));
            PTG_CUDA(cudaMemcpyAsync(grad + 2 * o, p.stage_out.as<double>() + 2 * o, c * 16, cudaMemcpyDeviceToHost,
                                     sout[b & 1]));
            rows_out = rows_ready;
        }
    }
    k_finalize<<<1, 256, 0, p.stream>>>(p.misfit.as<const double>(), N * p.misfit_per_pos, p.dotp.as<const double>(),
                                        v ? kPlaneBlocks : 0, p.value.as<double>());
    PTG_CHECK_LAUNCH();
    ++p.launches;
    PTG_CUDA(cudaEventRecord(ev_val, p.stream));
    PTG_CUDA(cudaStreamWaitEvent(p.s_out, ev_val, 0));
    PTG_CUDA(cudaMemcpyAsync(p.hval.p, p.value.p, sizeof(double), cudaMemcpyDeviceToHost, p.s_out));
    if (capture) {   // join the copy-out streams back into the capturing stream
        PTG_CUDA(cudaEventRecord(ev_join, p.s_out));
        PTG_CUDA(cudaStreamWaitEvent(p.stream, ev_join, 0));
        PTG_CUDA(cudaEventRecord(ev_join2, p.s_out2));
        PTG_CUDA(cudaStreamWaitEvent(p.stream, ev_join2, 0));
        return;
    }
    static const bool dbg = getenv("PTG_E2E_DEBUG") != nullptr;
    if (dbg) t_enq = std::chrono::steady_clock::now();
    PTG_CUDA(cudaStreamSynchronize(p.s_out2));
    PTG_CUDA(cudaStreamSynchronize(p.s_out));
    if (dbg) {
        const auto t_end = std::chrono::steady_clock::now();
        fprintf(stderr, "[e2e] enqueue %.1f us, wait %.1f us\n",
                std::chrono::duration<double, std::micro>(t_enq - t_beg).count(),
                std::chrono::duration<double, std::micro>(t_end - t_enq).count());
    }
    if (value) *value = *p.hval.as<double>();
}

// ------------------------------------------------- banded host eval (RMW)
// ptg_eval with host complex128 buffers on an RMW plan (configs 4-5): the
// object goes up in K row bands over two copy engines; the frames whose
// windows lie inside the rows uploaded so far run as one persistent RMW launch
// per band (launches are stream-ordered, so every earlier frame is complete
// when the next band's frames start -- the same summation order, bitwise the
// same gradient as plan_eval); gradient rows no pending frame touches go back
// (complex128) over the copy-out streams while later bands compute.  PCIe in,
// compute and PCIe out overlap instead of adding up.
static void eval_host_rmw(Plan& p, int metric, const double* z, double* value, double* grad) {
    using C = float2;
    const int n = p.n, w = p.w, N = p.N;
    const size_t nn = p.nn();
    const char* eb = getenv("PTG_RMW_BANDS");
    // config-5 ms per call (one copy stream per direction): 32 bands 26.4, 16: 26.8, 8: 28.6; unbanded 62.8
    const int K = eb ? std::max(1, std::min(64, atoi(eb))) : 32;
    const int H = (n + K - 1) / K;
    if (!p.s_in) {
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_in, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_out, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_in2, cudaStreamNonBlocking));
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_out2, cudaStreamNonBlocking));
    }
    // one stream per direction by default: with two H2D streams both copy
    // engines take the uploads queued up front and the downloads wait behind
    // them (PTG_E2E_STREAMS=2 restores two per direction, A/B)
    const char* es = getenv("PTG_E2E_STREAMS");
    const bool two = es && atoi(es) == 2;
    const cudaStream_t sin[2] = {p.s_in, two ? p.s_in2 : p.s_in}, sout[2] = {p.s_out, two ? p.s_out2 : p.s_out};
    while (p.ev_band.size() < (size_t)(2 * K + 4)) {
        cudaEvent_t e;
        PTG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p.ev_band.push_back(e);
    }
    cudaEvent_t* ev_in = p.ev_band.data();
    cudaEvent_t* ev_out = p.ev_band.data() + K;
    cudaEvent_t ev_start = p.ev_band[2 * K], ev_val = p.ev_band[2 * K + 1];
    p.zbuf.ensure(nn * sizeof(C));
    p.gbuf.ensure(nn * sizeof(C));
    p.stage.ensure(nn * 16);
    p.stage_out.ensure(nn * 16);
    double* st_z = p.stage.as<double>();
    C* zd = p.zbuf.as<C>();
    C* gd = p.gbuf.as<C>();
    const float* data = metric == PTG_DISTANCE ? p.amp.as<const float>() : p.inten.as<const float>();
    PTG_CUDA(cudaEventRecord(ev_start, p.stream));
    for (int i = 0; i < 2; ++i) {
        PTG_CUDA(cudaStreamWaitEvent(sin[i], ev_start, 0));
        PTG_CUDA(cudaStreamWaitEvent(sout[i], ev_start, 0));
    }
    for (int b = 0; b < K; ++b) {
        const size_t r0 = (size_t)std::min(n, b * H), r1 = (size_t)std::min(n, (b + 1) * H);
        if (r1 > r0)
            PTG_CUDA(cudaMemcpyAsync(st_z + 2 * r0 * n, z + 2 * r0 * n, (r1 - r0) * n * 16, cudaMemcpyHostToDevice,
                                     sin[b & 1]));
        PTG_CUDA(cudaEventRecord(ev_in[b], sin[b & 1]));
    }
    // gradient = 0, completion counters zeroed (no shift on this path)
    k_rmw_init<C><<<kRmwInitBlocks, 256, 0, p.stream>>>(nullptr, nullptr, gd, nn, nn, nullptr, p.rmw_done.as<unsigned>(),
                                                        N, p.rmw_work.as<unsigned>());
    PTG_CHECK_LAUNCH();
    ++p.launches;
    FrameArgs<float> a = frame_args<float>(p, zd, data);
    int k_cur = 0;
    size_t g = 0;        // row groups launched
    size_t rows_out = 0;
    for (int b = 0; b < K; ++b) {
        const int r0 = std::min(n, b * H), r1 = std::min(n, (b + 1) * H);
        PTG_CUDA(cudaStreamWaitEvent(p.stream, ev_in[b], 0));
        if (r1 > r0) dev_from_c128(PTG_C64, zd + (size_t)r0 * n, st_z + 2 * (size_t)r0 * n, (size_t)(r1 - r0) * n, p.stream);
        // whole row groups whose windows lie in the uploaded rows
        while (g < p.rmw_group_end.size() && (b == K - 1 || p.rmw_group_maxr0[g] + w <= r1)) ++g;
        const int k_end = g ? p.rmw_group_end[g - 1] : 0;
        if (k_end > k_cur) {
            PTG_CUDA(cudaMemsetAsync(p.rmw_work.p, 0, sizeof(unsigned), p.stream));
            if (metric == PTG_DISTANCE) launch_rmw<OP_DISTANCE>(p, a, data, gd, k_cur, k_end);
            else launch_rmw<OP_INTENSITY>(p, a, data, gd, k_cur, k_end);
            ++p.launches;
            k_cur = k_end;
        }
        // rows no pending frame touches are final
        const size_t ready = b == K - 1 ? (size_t)n : (size_t)std::min(p.rmw_sufmin_r0[k_cur], r1);
        if (ready > rows_out) {
            const size_t o = rows_out * n, c = (ready - rows_out) * n;
            dev_to_c128(PTG_C64, p.stage_out.as<double>() + 2 * o, gd + o, c, p.stream);
            PTG_CUDA(cudaEventRecord(ev_out[b], p.stream));
            PTG_CUDA(cudaStreamWaitEvent(sout[b & 1], ev_out[b], 0));
            PTG_CUDA(cudaMemcpyAsync(grad + 2 * o, p.stage_out.as<double>() + 2 * o, c * 16, cudaMemcpyDeviceToHost,
                                     sout[b & 1]));
            rows_out = ready;
        }
    }
    k_finalize<<<1, 256, 0, p.stream>>>(p.misfit.as<const double>(), N * p.misfit_per_pos, p.dotp.as<const double>(), 0,
                                        p.value.as<double>());
    PTG_CHECK_LAUNCH();
    ++p.launches;
    PTG_CUDA(cudaEventRecord(ev_val, p.stream));
    PTG_CUDA(cudaStreamWaitEvent(p.s_out, ev_val, 0));
    PTG_CUDA(cudaMemcpyAsync(p.hval.p, p.value.p, sizeof(double), cudaMemcpyDeviceToHost, p.s_out));
    PTG_CUDA(cudaStreamSynchronize(p.s_out2));
    PTG_CUDA(cudaStreamSynchronize(p.s_out));
    if (value) *value = *p.hval.as<double>();
}

static bool host_pinned(const void* ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void plan_eval_host(Plan& p, int metric, const double* z, const double* v, double* value, double* grad) {
    LaunchScope ls(p);
    plan_ensure(p, metric);
    if (p.rmw_mode && !p.comm && !v && grad && !p.timing &&
        !(getenv("PTG_NO_BANDED") && getenv("PTG_NO_BANDED")[0] == '1')) {
        eval_host_rmw(p, metric, z, value, grad);
        return;
    }
    static const bool off = getenv("PTG_NO_BANDED") && getenv("PTG_NO_BANDED")[0] == '1';   // A/B switch
    bool sorted = true;
    for (int j = 1; j < p.N && sorted; ++j) sorted = p.pos_h[2 * j] >= p.pos_h[2 * (j - 1)];
    const bool banded = !off && !p.comm && grad && p.planes_mode && p.chunks.size() == 1 && !p.mp && !p.timing && sorted &&
                        p.N > 0 && p.n >= 64;
    if (banded) {
        auto run = [&](bool capture) {
            if (p.prec == PTG_C64) eval_host_banded<float>(p, metric, z, v, value, grad, capture);
            else eval_host_banded<double>(p, metric, z, v, value, grad, capture);
        };
        static const bool nograph = getenv("PTG_NO_GRAPH") && getenv("PTG_NO_GRAPH")[0] == '1';   // A/B switch
        if (nograph || !host_pinned(z) || !host_pinned(grad) || (v && !host_pinned(v))) {
            run(false);
            return;
        }
        // one CUDA graph per pointer set: the ~30 copies, kernels and event
        // edges of the banded sequence cost ~90 us of host enqueue time
        // eagerly (longer than the PCIe transfers they schedule)
        auto key = [&] {
            return std::vector<const void*>{z, v, grad, (const void*)(intptr_t)metric, p.amp.p, p.inten.p, p.planes.p,
                                            p.zbuf.p, p.gbuf.p, p.vbuf.p, p.stage.p, p.stage_out.p, p.misfit.p,
                                            p.color.p, p.probe_epi.p, p.amp_cl.p, p.hval.p, p.value.p, p.dotp.p,
                                            p.counter.p};
        };
        if (p.hg.exec && key() == p.hg.key) {
            PTG_CUDA(cudaGraphLaunch(p.hg.exec, p.stream));
            p.launches += p.hg.launches;
            PTG_CUDA(cudaStreamSynchronize(p.stream));
            if (value) *value = *p.hval.as<double>();
            return;
        }
        if (key() != p.hg.seen) {   // first call with these pointers: eager
            run(false);
            p.hg.seen = key();
            return;
        }
        const int64_t l0 = p.launches;
        cudaGraph_t g = nullptr;
        PTG_CUDA(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
        try {
            run(true);
        } catch (...) {
            cudaStreamEndCapture(p.stream, &g);
            if (g) cudaGraphDestroy(g);
            p.launches = l0;
            throw;
        }
        PTG_CUDA(cudaStreamEndCapture(p.stream, &g));
        p.hg.launches = p.launches - l0;
        p.launches = l0;
        cudaGraphExec_t ex = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        PTG_CUDA(e);
        if (p.hg.exec) cudaGraphExecDestroy(p.hg.exec);
        p.hg.exec = ex;
        p.hg.key = key();
        PTG_CUDA(cudaGraphLaunch(p.hg.exec, p.stream));
        p.launches += p.hg.launches;
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        if (value) *value = *p.hval.as<double>();
        return;
    }
    const size_t bytes = p.nn() * p.celem();
    p.zbuf.ensure(bytes);
    p.gbuf.ensure(bytes);
    plan_upload_c128(p, z, p.zbuf.p);
    if (v) {
        p.vbuf.ensure(bytes);
        plan_upload_c128(p, v, p.vbuf.p);
    }
    plan_eval(p, metric, p.zbuf.p, v ? p.vbuf.p : nullptr, p.gbuf.p, p.value.as<double>());
    if (grad) plan_download_c128(p, p.gbuf.p, grad);
    const double val = plan_read_scalar(p, p.value.as<double>());
    if (value) *value = val;
}

// --------------------------------------------------------------- simulate
template <typename T>
static void simulate_t(Plan& p, const void* z) {
    FrameArgs<T> a = frame_args<T>(p, z, nullptr);
    a.data_out = p.inten.as<T>();
    for (auto& c : p.chunks) {
        if (c->count <= 0) continue;
        a.first = c->first;
        if (p.mp) {
            launch_mp<T, OP_SIMULATE>(p, a, c->first, c->count, 3);
        } else {
            launch_frame_m<T, OP_SIMULATE>(p.M, a, c->count, p.stream);
            ++p.launches;
        }
    }
}

void plan_simulate(Plan& p, const void* z) {
    LaunchScope ls(p);
    const size_t len = (size_t)p.N * p.MM();
    p.inten.ensure(std::max<size_t>(1, len) * p.relem());
    if (p.prec == PTG_C64) simulate_t<float>(p, z);
    else simulate_t<double>(p, z);
    p.inten_valid = true;
    p.amp_valid = false;
    plan_refresh_amp(p);
}

// ---------------------------------------------------------------- project
template <typename T>
__global__ void k_roll(const cplx<T>* __restrict__ in, int M, int r0, int c0, cplx<T>* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M * M; i += gridDim.x * blockDim.x) {
        const int r = i / M, c = i % M;
        out[(size_t)((r + r0) % M) * M + (c + c0) % M] = in[i];
    }
}

template <typename T>
static void project_t(Plan& p, const void* z, int k, void* out) {
    FrameArgs<T> a = frame_args<T>(p, z, p.amp.as<const T>());
    p.frame.ensure(p.MM() * p.celem() * 2);
    a.first = k;
    a.frame_out = p.frame.as<cplx<T>>() - (size_t)k * p.MM();
    if (p.mp) {
        launch_mp<T, OP_PROJECT>(p, a, k, 1);
    } else {
        launch_frame_m<T, OP_PROJECT>(p.M, a, 1, p.stream);
        ++p.launches;
    }
    // ref mode: return the projection in object coordinates (objectives.cpp:42-50)
    const int r0 = p.ref_mode() ? p.pos_h[2 * k] : 0, c0 = p.ref_mode() ? p.pos_h[2 * k + 1] : 0;
    k_roll<T><<<grid_for(p.MM()), 256, 0, p.stream>>>(p.frame.as<const cplx<T>>(), p.M, r0, c0,
                                                       static_cast<cplx<T>*>(out));
    PTG_CHECK_LAUNCH();
    ++p.launches;
}

void plan_project(Plan& p, const void* z, int k, void* out) {
    LaunchScope ls(p);
    if (k < 0 || k >= p.N) raise(PTG_ERR_DOMAIN, "pattern index out of range");
    plan_ensure(p, PTG_DISTANCE);
    if (p.prec == PTG_C64) project_t<float>(p, z, k, out);
    else project_t<double>(p, z, k, out);
}

// ------------------------------------------------------------------ fft2
// fft2 / ifft2 (field.hpp:91-93, kernels.cpp:34-85) of one n x n complex128
// field on the device: the objective kernels' own 2-D FFT (single-CTA frame
// kernel, n <= 64 in complex128)
void dev_fft2(const void* in, int n, bool inverse, void* out, cudaStream_t s) {
    if (!is_pow2(n)) raise(PTG_ERR_GEOMETRY, "fft2: grid side must be a positive power of two, got " + std::to_string(n));
    if (!frame_single_cta(PTG_C128, n))
        raise(PTG_ERR_CONFIG, "fft2: n=" + std::to_string(n) + " exceeds the single-CTA complex128 transform (n <= 64)");
    DevMem pos;
    pos.alloc(sizeof(int2));
    PTG_CUDA(cudaMemsetAsync(pos.p, 0, sizeof(int2), s));
    FrameArgs<double> a{};
    a.z = static_cast<const double2*>(in);
    a.pos = pos.as<const int2>();
    a.frame_out = static_cast<double2*>(out);
    a.n = n;
    a.w = n;
    a.first = 0;
    if (inverse) launch_frame_m<double, OP_FFT_INV>(n, a, 1, s);
    else launch_frame_m<double, OP_FFT_FWD>(n, a, 1, s);
    count_launch();
    PTG_CUDA(cudaStreamSynchronize(s));   // `pos` is freed on return
}

// -------------------------------------------------------------------- PIE
// z_win += weight o (Pi(psi) - psi) for one position (multi-pass frames)
template <typename T>
__global__ void k_pie_update(cplx<T>* __restrict__ z, const cplx<T>* __restrict__ proj,
                             const cplx<T>* __restrict__ probe, int r0, int c0, int n, int w, int M,
                             const cplx<T>* __restrict__ wgt, T damping) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w * w; idx += gridDim.x * blockDim.x) {
        const int r = idx / w, c = idx % w;
        cplx<T>* zp = z + (size_t)(r0 + r) * n + (c0 + c);
        const cplx<T> zz = *zp;
        const cplx<T> psi = probe ? cmul(probe[(size_t)r * M + c], zz) : zz;
        const cplx<T> dl = csub(proj[(size_t)r * M + c], psi);
        *zp = cadd(zz, wgt ? cmul(wgt[idx], dl) : cscale(dl, damping));
    }
}

template <typename T>
static void pie_sweep_mp(Plan& p, void* z, const void* wgt, double damping) {
    p.frame.ensure(p.MM() * p.celem() * 2 + (size_t)p.w * p.w * p.celem());
    FrameArgs<T> a = frame_args<T>(p, z, p.amp.as<const T>());
    for (int k = 0; k < p.N; ++k) {
        a.first = k;
        a.frame_out = p.frame.as<cplx<T>>() - (size_t)k * p.MM();
        launch_mp<T, OP_PROJECT>(p, a, k, 1);
        k_pie_update<T><<<grid_for((size_t)p.w * p.w), 256, 0, p.stream>>>(
            static_cast<cplx<T>*>(z), p.frame.as<const cplx<T>>(), p.has_probe ? p.probe.as<const cplx<T>>() : nullptr,
            p.pos_h[2 * k], p.pos_h[2 * k + 1], p.n, p.w, p.M, static_cast<const cplx<T>*>(wgt), (T)damping);
        PTG_CHECK_LAUNCH();
        ++p.launches;
    }
}

void plan_pie_sweep(Plan& p, void* z, double gamma) {
    LaunchScope ls(p);
    if (gamma < 0.0) raise(PTG_ERR_CONFIG, "pie: gamma must be non-negative");
    plan_ensure(p, PTG_DISTANCE);
    if (p.N == 0) return;
    const void* wgt = nullptr;
    if (p.has_probe) {
        // Alg. 1 weight: (|P|/max|P|) conj(P) / (|P|^2 + gamma), on the window
        const int w = p.w, M = p.M;
        double pmax = 0.0;
        for (size_t i = 0; i < p.MM(); ++i) pmax = std::max(pmax, std::hypot(p.probe_h[2 * i], p.probe_h[2 * i + 1]));
        std::vector<double> wg(2 * (size_t)w * w);
        for (int r = 0; r < w; ++r)
            for (int c = 0; c < w; ++c) {
                const double* P = &p.probe_h[2 * ((size_t)r * M + c)];
                const double a = std::hypot(P[0], P[1]);
                const double s = (pmax > 0.0 ? a / pmax : 0.0) / (a * a + gamma);
                wg[2 * ((size_t)r * w + c)] = s * P[0];
                wg[2 * ((size_t)r * w + c) + 1] = -s * P[1];
            }
        p.stage.ensure(wg.size() * sizeof(double));
        p.frame.ensure(p.MM() * p.celem() * 2 + (size_t)w * w * p.celem());
        void* dw = static_cast<char*>(p.frame.p) + p.MM() * p.celem() * 2;
        PTG_CUDA(cudaMemcpyAsync(p.stage.p, wg.data(), wg.size() * sizeof(double), cudaMemcpyHostToDevice, p.stream));
        dev_from_c128(p.prec, dw, p.stage.as<double>(), (size_t)w * w, p.stream);
        wgt = dw;
    }
    const double damping = 1.0 / (1.0 + gamma);
    if (p.mp) {   // frames beyond one CTA: per position, project (3 passes) then update
        if (p.prec == PTG_C64) pie_sweep_mp<float>(p, z, wgt, damping);
        else pie_sweep_mp<double>(p, z, wgt, damping);
        return;
    }
    if (p.prec == PTG_C64) launch_pie<float>(p, z, wgt, damping);
    else launch_pie<double>(p, z, wgt, damping);
}

// ------------------------------------------------------------- coarsening
// buildCoarseLevel (multigrid.cpp:79-93) restated for the patch model:
// n/2, M/2, w/2, floor(pos/2), probe -> restrictField(probe), data ->
// restrictData, all on device.
std::unique_ptr<Plan> plan_coarsen(Plan& f) {
    if (f.n < 16) raise(PTG_ERR_GEOMETRY, "buildCoarseLevel: refuse to coarsen below n = 8");
    if (f.w < 2 || f.w % 2 != 0)
        raise(PTG_ERR_GEOMETRY, "buildCoarseLevel: window size must be even and >= 2, got " + std::to_string(f.w));
    if (f.M < 4 || f.M % 4 != 0) raise(PTG_ERR_GEOMETRY, "restrictData: grid side must be a multiple of 4");
    LaunchScope ls(f);
    std::vector<int32_t> pos(f.pos_h.size());
    for (size_t i = 0; i < pos.size(); ++i) pos[i] = f.pos_h[i] / 2;
    std::vector<double> probe;
    if (f.has_probe) {
        probe.resize(2 * (size_t)(f.M / 2) * (f.M / 2));
        const int M = f.M, MH = M / 2;
        for (int r = 0; r < MH; ++r)
            for (int c = 0; c < MH; ++c)
                for (int q = 0; q < 2; ++q) {
                    const double a = f.probe_h[2 * ((size_t)(2 * r) * M + 2 * c) + q];
                    const double b = f.probe_h[2 * ((size_t)(2 * r) * M + 2 * c + 1) + q];
                    const double cc = f.probe_h[2 * ((size_t)(2 * r + 1) * M + 2 * c) + q];
                    const double d = f.probe_h[2 * ((size_t)(2 * r + 1) * M + 2 * c + 1) + q];
                    probe[2 * ((size_t)r * MH + c) + q] = ((a + b) + (cc + d)) * 0.25;
                }
    }
    ptg_plan_desc d{};
    d.n = f.n / 2;
    d.M = f.M / 2;
    d.w = f.w / 2;
    d.N = f.N;
    d.positions = pos.data();
    d.probe = f.has_probe ? probe.data() : nullptr;
    d.data = nullptr;
    d.precision = f.prec;
    d.device = f.device;
    auto c = plan_create(d);
    // restrictData on device: intensities x 1/16 (or amplitudes x 1/4)
    const size_t len = (size_t)c->N * c->MM();
    const int dt = f.prec == PTG_C64 ? PTG_F32 : PTG_F64;
    if (f.inten_valid) {
        c->inten.ensure(std::max<size_t>(1, len) * c->relem());
        PTG_CUDA(cudaStreamSynchronize(f.stream));
        if (len) dev_restrict_data(dt, f.inten.p, f.N, f.M, c->inten.p, 1.0 / 16.0, c->stream);
        c->inten_valid = true;
        plan_refresh_amp(*c);
    } else if (f.amp_valid) {
        c->amp.ensure(std::max<size_t>(1, len) * c->relem());
        PTG_CUDA(cudaStreamSynchronize(f.stream));
        if (len) dev_restrict_data(dt, f.amp.p, f.N, f.M, c->amp.p, 0.25, c->stream);
        c->amp_valid = true;
    } else {
        raise(PTG_ERR_CONFIG, "coarsen: fine plan has no data");
    }
    PTG_CUDA(cudaStreamSynchronize(c->stream));
    return c;
}

// ------------------------------------------------------------ host helpers
void plan_upload_c128(Plan& p, const double* host, void* dev) {
    if (p.prec == PTG_C128) {
        PTG_CUDA(cudaMemcpyAsync(dev, host, p.nn() * 16, cudaMemcpyHostToDevice, p.stream));
        return;
    }
    p.stage.ensure(p.nn() * 16);
    PTG_CUDA(cudaMemcpyAsync(p.stage.p, host, p.nn() * 16, cudaMemcpyHostToDevice, p.stream));
    LaunchScope ls(p);
    dev_from_c128(p.prec, dev, p.stage.as<double>(), p.nn(), p.stream);
}

void plan_download_c128(Plan& p, const void* dev, double* host) {
    if (p.prec == PTG_C128) {
        PTG_CUDA(cudaMemcpyAsync(host, dev, p.nn() * 16, cudaMemcpyDeviceToHost, p.stream));
        return;
    }
    p.stage.ensure(p.nn() * 16);
    LaunchScope ls(p);
    dev_to_c128(p.prec, p.stage.as<double>(), dev, p.nn(), p.stream);
    PTG_CUDA(cudaMemcpyAsync(host, p.stage.p, p.nn() * 16, cudaMemcpyDeviceToHost, p.stream));
}

double plan_read_scalar(Plan& p, const double* dev) {
    PTG_CUDA(cudaMemcpyAsync(p.hval.p, dev, sizeof(double), cudaMemcpyDeviceToHost, p.stream));
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    return *p.hval.as<double>();
}

bool plan_nonfinite(Plan& p, const void* x, size_t len) {
    LaunchScope ls(p);
    dev_nonfinite(p.prec, x, len, p.flag.as<int>(), p.stream);
    int f = 0;
    PTG_CUDA(cudaMemcpyAsync(&f, p.flag.p, sizeof(int), cudaMemcpyDeviceToHost, p.stream));
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    return f != 0;
}

double plan_dot(Plan& p, const void* a, const void* b, size_t len) {
    LaunchScope ls(p);
    dev_dot(p.prec, a, b, len, p.scratch.as<double>(), p.value.as<double>() + 1, p.stream);
    return plan_read_scalar(p, p.value.as<double>() + 1);
}

}  // namespace ptg

#ifdef ABL_TIMELINE
extern "C" int ptg_debug_timeline(void* dst, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(dst, ptg::g_tl, bytes < sizeof(ptg::g_tl) ? bytes : sizeof(ptg::g_tl));
}
extern "C" int ptg_debug_rmw_timeline(void* dst, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(dst, ptg::g_rmw_tl, bytes < sizeof(ptg::g_rmw_tl) ? bytes : sizeof(ptg::g_rmw_tl));
}
#endif
