// hyg_api.cu — host runtime behind include/hygro_b200.h.
//
// A context owns the device-resident state of one model (a batch of walls on
// one grid, optionally coupled to zones) and plays the role of the
// reference's BuildingModel + BuildingState + run() (building.hpp:38-102):
//   * independent exterior walls with constant coefficients on a grid that
//     tiles onto lanes  -> K1 (k_coupled.cuh), many steps fused per launch;
//   * everything else (zones, analytic coefficients, any N) -> the one-step
//     kernels of k_step.cuh, one launch per step (+ one zone launch).
// Forcing signals are evaluated on the host per time layer exactly as
// Signal::operator() (signal.hpp:39-50) at the accumulated time t
// (BuildingState::t, building.cpp:185), and uploaded as per-layer tables.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/hygro_b200.h"
#include "k_coupled.cuh"
#include "k_step.cuh"
#include "k_nonlinear.cuh"
#include "k_dv_warp.cuh"
#include "k_material.cuh"
#include "k_ring.cuh"
#include "k_ring_reg.cuh"
#include "k_ring_pipe.cuh"
#include "k_ring_split.cuh"

using namespace hyg;

namespace {

constexpr int kChunk = 128;     // forcing rows staged per shared-memory chunk
constexpr int kRingS = 8;       // K4: steps per launch (halo depth S-1 zones)
#ifndef HYG_RING_REG_S
#define HYG_RING_REG_S 8
#endif
constexpr int kRingRegS = HYG_RING_REG_S;   // K4r: steps per launch (S = 9 measured 3.12e11 vs 3.49e11 at 8: spills)
#ifndef HYG_RING_PIPE_S
#define HYG_RING_PIPE_S 12
#endif
constexpr int kRingPipeS = HYG_RING_PIPE_S; // K5: steps per launch
#ifndef HYG_RING_SPLIT_S
#define HYG_RING_SPLIT_S 8
#endif
#ifndef HYG_RING_AUTO
#define HYG_RING_AUTO 4
#endif
constexpr int kRingAuto = HYG_RING_AUTO;         // the zone-ring kernel HYG_TUNE_RING_KERNEL = 0 selects (4: K6, 1: K4r)
constexpr int kRingSplitS = HYG_RING_SPLIT_S;   // K6 (k_ring_split.cuh): steps per cone launch
#ifndef HYG_RING_SPLIT_M
#define HYG_RING_SPLIT_M 2
#endif
constexpr int kRingSplitM = HYG_RING_SPLIT_M;   // K6: cone launches per walls launch (walls march M x S steps), default
constexpr int kRingSplitMaxM = 3;
constexpr int kWarps = 4;       // warps per CTA of K1

struct SigHost {
    hyg_signal s{};
    std::vector<hyg_window> win;
    void set(const hyg_signal& x) {
        s = x;
        win.assign(x.windows, x.windows + (x.windows ? x.n_windows : 0));
        s.n_windows = static_cast<int32_t>(win.size());
        s.windows = nullptr;
    }
    double operator()(double t) const {   // signal.hpp:39-50
        double v = s.base;
        if (s.form == HYG_SIG_SIN) {
            v += s.amplitude * std::sin(2.0 * M_PI * (t - s.phase) / s.period);
        } else if (s.form == HYG_SIG_SIN2) {
            const double x = std::sin(2.0 * M_PI * (t - s.phase) / s.period);
            v += s.amplitude * x * x;
        }
        for (const auto& w : win)
            if (t >= w.from && t < w.to) v += w.value;
        return v;
    }
};

struct ChannelHost {
    SigHost u, v, g, q;
    int64_t tab_first = 0;
    std::vector<hyg_ambient> tab;   // explicit per-layer override
    bool flux_free() const {        // g and q identically zero: K1 without flux terms
        auto zero = [](const SigHost& s) {
            if (s.s.form != HYG_SIG_CONSTANT || s.s.base != 0.0) return false;
            for (const auto& w : s.win)
                if (w.value != 0.0) return false;
            return true;
        };
        if (!zero(g) || !zero(q)) return false;
        for (const auto& a : tab)
            if (a.g_inf != 0.0 || a.q_inf != 0.0) return false;
        return true;
    }
    Ambient at(int64_t layer, double t) const {
        if (!tab.empty() && layer >= tab_first && layer < tab_first + static_cast<int64_t>(tab.size())) {
            const hyg_ambient& a = tab[layer - tab_first];
            return Ambient{a.u_inf, a.v_inf, a.g_inf, a.q_inf};
        }
        return Ambient{u(t), v(t), g(t), q(t)};
    }
};

// explicit per-layer values (zone sources: 3 per layer, outdoor: 2 per layer)
struct TableHost {
    int64_t first = 0;
    int width = 1;
    std::vector<double> v;
    bool covers(int64_t L) const {
        return !v.empty() && L >= first && L < first + static_cast<int64_t>(v.size() / width);
    }
};

struct Pending { int stat; cudaEvent_t e0, e1; double updates; };
struct Stat { std::string name; int64_t launches = 0; double ms = 0, updates = 0; };

void set_status(hyg_status* st, int code, const char* msg) {
    if (!st) return;
    st->code = code;
    std::snprintf(st->message, sizeof st->message, "%s", msg);
}

void clear_status(hyg_status* st) {
    if (!st) return;
    std::memset(st, 0, sizeof *st);
    st->wall = -1;
    st->zone = -1;
    st->layer = -1;
}

}  // namespace

struct hyg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;       // the stream every launch and copy goes to
    cudaStream_t own_stream = nullptr;   // the context's own (hyg_set_stream(NULL) restores it)
    // model
    int n_walls = 0, n = 0;
    double dx = 0;
    int precision = HYG_F64, coeff_kind = HYG_COEFF_CONSTANT;
    double p[4] = {0, 0, 0, 0};
    std::vector<Groups> groups;
    std::vector<Biot> biot;
    std::vector<Attach> attach;
    std::vector<ChannelHost> channels;
    std::vector<ZoneDev> zones;
    std::vector<ZoneLinkDev> zlinks;
    std::vector<InzLinkDev> inz;
    std::vector<SigHost> zsrc;    // [n_sources*3]: g_o, q_o, q_h
    SigHost out_u, out_v;
    std::vector<TableHost> src_tab;   // [n_sources] overrides (hyg_set_source_table)
    TableHost out_tab;                // outdoor override (hyg_set_outdoor_table)
    double dt = 1e-3, norm = 1e3, eta_factor = 1e-2;
    int max_subiters = 100;
    // device state (ping-pong)
    double* s64[2][4] = {};
    float* s32[2][4] = {};
    int cur = 0;
    double* zu[2] = {};
    double* zv[2] = {};
    int zcur = 0;
    void* snap[4] = {};          // hyg_snapshot buffers (allocated on first use)
    double* snap_z[2] = {};
    double snap_t = 0.0;
    int64_t snap_layer = -1;
    Groups* d_groups = nullptr;
    Biot* d_biot = nullptr;
    Attach* d_attach = nullptr;
    int* d_chan = nullptr;
    WallCoef* d_coef = nullptr;
    double coef_dt = -1.0;
    ZoneDev* d_zones = nullptr;
    ZoneLinkDev* d_zlinks = nullptr;
    InzLinkDev* d_inz = nullptr;
    Ambient* d_table = nullptr;
    size_t table_cap = 0;
    std::vector<Ambient> h_table;
    Ambient* d_boot = nullptr;     // ambient row of the starting step
    std::vector<Ambient> h_boot;
    bool tab_valid = false;        // cache key of the table on the device
    int64_t tab_layer0 = 0;
    size_t tab_rows = 0;
    uint64_t tab_gen = 0, gen = 0; // gen bumps on hyg_set_channel_table
    double tab_t0 = 0, tab_t1 = 0;
    double* d_src = nullptr;
    size_t src_cap = 0;
    std::vector<double> h_src;
    int* d_flag = nullptr;
    unsigned long long* d_key = nullptr;
    // shard ownership (hyg_set_owned): guard/residual ranges and the reduction
    int64_t own_c0 = 0, own_c1 = INT64_MAX;
    int own_z0 = 0, own_z1 = INT32_MAX;
    hyg_reduce_fn reduce = nullptr;
    void* reduce_user = nullptr;
    // time
    double t = 0.0;
    int64_t layer = 0;
    // dispatch
    bool fused = false;        // K1: constant exterior walls on a fused grid
    bool nl_fused = false;     // K2: analytic d(v) exterior walls, n <= 1024
    bool tiled = false;        // K3: one long analytic d(v) exterior wall, n > 1024
    TiledMaps tmaps[2];        // K3w: tensor maps of the state arrays s64[b][0..3] (rows of 8 nodes, 64-byte swizzle)
    bool tmaps_ok = false;     // cuTensorMapEncodeTiled succeeded for all eight
    // hyg_advance_overlapped (one-shot, consumed by the next K3w launch): the windows reading
    // none of the first ov_lo / last ov_hi cells go first, the rest waits for ov_event
    int64_t ov_lo = 0, ov_hi = 0;
    cudaEvent_t ov_event = nullptr;
    cudaStream_t xstream = nullptr;   // hyg_set_exchange_stream: pack / unpack run here (nullptr: on `stream`)
    int tiled_load = 0;        // HYG_TUNE_TILED_LOAD: 0 TMA tiles (k_dv_tiled_tma), 1 cp.async (k_dv_tiled_stream)
    bool fo_m_pos = true;      // every wall has Fo_M > 0 (K2/K3 scale by 2 Fo_M dt/dx^2)
    bool flux = true;
    int seg_len = 4096;
    // measurement
    cudaEvent_t ev[16] = {};
    bool profiling = false;
    std::vector<Pending> pending;
    std::vector<Stat> stats;
    int64_t launches = 0;

    // state-dependent coefficients (per-wall CoefficientModel) and radiation
    std::vector<int> wall_kind;      // kCoeff* per wall
    bool any_nonlinear = false, any_material = false;
    double T_i = 293.15, P_vi = 0.0;
    int* d_wall_kind = nullptr;
    mat::Set* d_ref = nullptr;       // reference sets of material walls
    double* d_star = nullptr;        // StarTables scratch [9][cells] (allocated on first use)
    double* d_impl = nullptr;        // implicit start scratch (allocated on first use)
    unsigned long long* d_dom = nullptr;
    bool has_rad = false;
    bool ring = false;               // K4: zone-ring temporal blocking applies
    int ring_W = 0, ring_B = 0;
    int ring_reg_B = 0;              // K4r (registers + prefetch): zones per CTA, 0 if not applicable
    int ring_grid_cap = 0;           // HYG_TUNE_RING_GRID: K4r/K5 persistent grid cap (0: one CTA per SM)
    int ring_pipe_B = 0;             // K5 (k_ring_pipe.cuh): zones per block, 0 if not applicable
    int ring_kernel = 0;             // HYG_TUNE_RING_KERNEL: 0 auto (K6), 1 K4r, 2 K4, 3 K5, 4 K6
    int ring_cone_LB = 0;            // K6 phase 1: local zones per CTA (owned + 2 S halo), 0 if not applicable
    double* d_ring_rowsT = nullptr;  // K6 phase 1: cone rows transposed [12][walls] for rows_dt (k_ring_cone_rows)
    double* d_ring_zpT = nullptr;    // K6 phase 1: the zone parameter blocks transposed [kRingZP][zones]
    double rows_dt = -1.0;
    int ring_split_m = kRingSplitM;  // HYG_TUNE_RING_DEPTH: cone launches (of kRingSplitS steps) per walls launch, 1..3
    double* d_ring_tail[2][4] = {};  // K6: compact tails between the cone launches of one walls launch (k_ring_stub)
    double* d_ring_zt[2][2] = {};    // K6: zone air between those cone launches [buffer][u, v]
    double* d_ring_series = nullptr; // K6: layer-k air of every zone for the S steps of a launch [zones][S][2]
    bool mat_exact = false;          // HYG_TUNE_MATERIAL_EXACT: CrMath evaluation + IEEE-division rows
    bool owned_partial = false;      // hyg_set_owned narrowed the guard to a shard's range
    int ring_dbg_skip = 0;           // HYG_DEBUG_RING_SKIP (timing experiments only; wrong results)
    double* d_ring_zp = nullptr;     // K4r per-zone parameter blocks [zones][kRingZP]
    bool ring_reg_small = false;     // every zone: <= 6 wall links, <= 2 ring peers
    int rad_groups = 0, rad_terms = 0;
    int *d_rad_tgt = nullptr, *d_rad_grp = nullptr;
    double *d_rad_num = nullptr, *d_rad_den = nullptr, *d_rad_coef = nullptr, *d_qrad = nullptr;
    int64_t *d_rad_e = nullptr, *d_rad_r = nullptr;

    int64_t cells() const { return static_cast<int64_t>(n_walls) * n; }
};

#define HYG_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            char m_[200];                                                               \
            std::snprintf(m_, sizeof m_, "CUDA error %s at %s:%d", cudaGetErrorString(e_), \
                          __FILE__, __LINE__);                                          \
            set_status(status, HYG_ECUDA, m_);                                          \
            return HYG_ECUDA;                                                           \
        }                                                                               \
    } while (0)

namespace {

int stat_index(hyg_ctx* c, const char* name) {
    for (size_t i = 0; i < c->stats.size(); ++i)
        if (c->stats[i].name == name) return static_cast<int>(i);
    c->stats.push_back(Stat{name});
    return static_cast<int>(c->stats.size() - 1);
}

// bracket one launch with events when profiling is on
struct LaunchScope {
    hyg_ctx* c;
    Pending p{};
    bool on;
    LaunchScope(hyg_ctx* ctx, const char* name, double updates) : c(ctx), on(ctx->profiling) {
        ++c->launches;
        if (!on) return;
        p.stat = stat_index(c, name);
        p.updates = updates;
        cudaEventCreate(&p.e0);
        cudaEventCreate(&p.e1);
        cudaEventRecord(p.e0, c->stream);
    }
    ~LaunchScope() {
        if (!on) return;
        cudaEventRecord(p.e1, c->stream);
        c->pending.push_back(p);
    }
};

void drain_pending(hyg_ctx* c) {
    for (auto& p : c->pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.e1);
        cudaEventElapsedTime(&ms, p.e0, p.e1);
        Stat& s = c->stats[p.stat];
        s.launches += 1;
        s.ms += ms;
        s.updates += p.updates;
        cudaEventDestroy(p.e0);
        cudaEventDestroy(p.e1);
    }
    c->pending.clear();
}

// halo payloads: cells [c0, c0+count) of the four layers <-> buf[4][count]
struct Layers4 { double* p[4]; };
__global__ void k_pack_cells(Layers4 L, int64_t c0, int64_t count, double* buf) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < 4 * count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int f = static_cast<int>(i / count);
        buf[i] = L.p[f][c0 + (i - f * count)];
    }
}
__global__ void k_unpack_cells(Layers4 L, int64_t c0, int64_t count, const double* buf) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < 4 * count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int f = static_cast<int>(i / count);
        L.p[f][c0 + (i - f * count)] = buf[i];
    }
}

// ---- per-device launch attributes ----------------------------------------------
// cudaFuncSetAttribute and the SM count are per device: every kernel keeps a
// bit per device (set under a lock) instead of a process-wide "done" flag, so
// contexts on several GPUs of one process each configure their own device
constexpr int kMaxDevices = 64;
std::mutex g_attr_mu;

template <typename K>
void ensure_smem_attr(K kernel, int device, int bytes) {
    static std::unordered_map<const void*, unsigned long long> done;   // kernel -> device mask
    std::lock_guard<std::mutex> lk(g_attr_mu);
    const unsigned long long bit = 1ull << (device & (kMaxDevices - 1));
    unsigned long long& m = done[reinterpret_cast<const void*>(kernel)];
    if (m & bit) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    m |= bit;
}

int sm_count(int device) {
    static int n[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& x = n[device & (kMaxDevices - 1)];
    if (!x) cudaDeviceGetAttribute(&x, cudaDevAttrMultiProcessorCount, device);
    return std::max(x, 1);
}

// ---- tensor maps (driver entry point through the runtime: libcuda is not linked) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// a state array of n fp64 nodes as rows of 8 nodes (64 B), boxes of 32 rows (one K3w
// window), 64-byte swizzle (k_dv_tiled_tma)
bool make_row_map(CUtensorMap* m, double* base, int64_t n) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || n < 8 * 32) return false;
    const cuuint64_t dims[2] = {8, static_cast<cuuint64_t>(n / 8)};
    const cuuint64_t strides[1] = {64};
    const cuuint32_t box[2] = {8, 32};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- K1 dispatch -------------------------------------------------------------
template <typename Real>
using SegFn = void (*)(const CoupledSegArgs<Real>&, int grid, int smem, cudaStream_t, int device);

template <typename Real, int LPW, int NPT, bool FLUX, bool EXACT>
void launch_seg(const CoupledSegArgs<Real>& a, int grid, int smem, cudaStream_t s, int device) {
    auto k = k_df_coupled<Real, LPW, NPT, kWarps, kChunk, FLUX, EXACT>;
    ensure_smem_attr(k, device, 64 * 1024);
    k<<<grid, kWarps * 32, smem, s>>>(a);
}

template <typename Real, int LPW, int NPT>
SegFn<Real> pick4(bool flux, bool exact) {
    if (flux) return exact ? launch_seg<Real, LPW, NPT, true, true> : launch_seg<Real, LPW, NPT, true, false>;
    return exact ? launch_seg<Real, LPW, NPT, false, true> : launch_seg<Real, LPW, NPT, false, false>;
}

// supported fused grids: N = LPW * NPT
template <typename Real>
SegFn<Real> pick_seg(int n, bool flux, bool exact, int* lpw) {
    switch (n) {
        case 64: *lpw = 16; return pick4<Real, 16, 4>(flux, exact);
        case 128: *lpw = 16; return pick4<Real, 16, 8>(flux, exact);
        case 256:
            // fp32 (configs[2]): 8 lanes x 32 nodes issues fewer shuffles/selects
            // per update, +6 % over 16 x 16 (profiles/r01_k1_variants.txt)
            if (sizeof(Real) == 4) {
                *lpw = 8;
                return pick4<Real, 8, 32>(flux, exact);
            }
            *lpw = 16;
            return pick4<Real, 16, 16>(flux, exact);
        case 512: *lpw = 32; return pick4<Real, 32, 16>(flux, exact);
        default: return nullptr;
    }
}

bool fused_grid(int n) { return n == 64 || n == 128 || n == 256 || n == 512; }

// ---- forcing tables ---------------------------------------------------------------
// rows for layers [layer0, layer0 + rows), row k evaluated at time times[k]
int upload_table(hyg_ctx* c, int64_t layer0, const std::vector<double>& times, hyg_status* status) {
    const size_t rows = times.size();
    const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
    // the device copy is reused when the same layers at the same times were
    // uploaded last (repeated runs from a snapshot)
    if (c->tab_valid && c->tab_layer0 == layer0 && c->tab_rows == rows && c->tab_gen == c->gen &&
        c->tab_t0 == times.front() && c->tab_t1 == times.back())
        return HYG_OK;
    c->tab_valid = true;
    c->tab_layer0 = layer0;
    c->tab_rows = rows;
    c->tab_gen = c->gen;
    c->tab_t0 = times.front();
    c->tab_t1 = times.back();
    c->h_table.resize(rows * nch);
    for (size_t k = 0; k < rows; ++k)
        for (int ch = 0; ch < static_cast<int>(c->channels.size()); ++ch)
            c->h_table[k * nch + ch] = c->channels[ch].at(layer0 + static_cast<int64_t>(k), times[k]);
    if (c->channels.empty())
        for (size_t k = 0; k < rows; ++k) c->h_table[k] = Ambient{1, 1, 0, 0};
    const size_t bytes = rows * nch * sizeof(Ambient);
    if (bytes > c->table_cap) {
        if (c->d_table) cudaFree(c->d_table);
        HYG_CUDA(cudaMalloc(&c->d_table, bytes));
        c->table_cap = bytes;
    }
    HYG_CUDA(cudaMemcpyAsync(c->d_table, c->h_table.data(), bytes, cudaMemcpyHostToDevice, c->stream));
    // the host vector must outlive the async copy
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

// zone sources + outdoor per step: [rows][n_src*3 + 2]
// zone sources + outdoor, rows for layers [layer0, layer0 + times.size())
int upload_src(hyg_ctx* c, int64_t layer0, const std::vector<double>& times, hyg_status* status) {
    const int nsrc = static_cast<int>(c->zsrc.size() / 3);
    const int w = nsrc * 3 + 2;
    c->h_src.resize(times.size() * w);
    for (size_t k = 0; k < times.size(); ++k) {
        const int64_t L = layer0 + static_cast<int64_t>(k);
        double* r = &c->h_src[k * w];
        for (int s = 0; s < nsrc; ++s) {
            const TableHost& tb = c->src_tab[s];
            if (tb.covers(L)) {
                for (int i = 0; i < 3; ++i) r[3 * s + i] = tb.v[(L - tb.first) * 3 + i];
            } else {
                for (int i = 0; i < 3; ++i) r[3 * s + i] = c->zsrc[3 * s + i](times[k]);
            }
        }
        if (c->out_tab.covers(L)) {
            r[nsrc * 3 + 0] = c->out_tab.v[(L - c->out_tab.first) * 2 + 0];
            r[nsrc * 3 + 1] = c->out_tab.v[(L - c->out_tab.first) * 2 + 1];
        } else {
            r[nsrc * 3 + 0] = c->out_u(times[k]);
            r[nsrc * 3 + 1] = c->out_v(times[k]);
        }
    }
    const size_t bytes = c->h_src.size() * sizeof(double);
    if (bytes > c->src_cap) {
        if (c->d_src) cudaFree(c->d_src);
        HYG_CUDA(cudaMalloc(&c->d_src, bytes));
        c->src_cap = bytes;
    }
    HYG_CUDA(cudaMemcpyAsync(c->d_src, c->h_src.data(), bytes, cudaMemcpyHostToDevice, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

StepArgs step_args(hyg_ctx* c, int from, double dt) {
    StepArgs a{};
    a.n_walls = c->n_walls;
    a.n = c->n;
    a.dx = c->dx;
    a.dt = dt;
    a.groups = c->d_groups;
    a.biot = c->d_biot;
    a.attach = c->d_attach;
    a.n_channels = std::max<int>(1, static_cast<int>(c->channels.size()));
    a.zu = c->zu[c->zcur];
    a.zv = c->zv[c->zcur];
    a.coeff_kind = c->coeff_kind == HYG_COEFF_ANALYTIC_D ? kCoeffAnalyticD : kCoeffConstant;
    for (int i = 0; i < 4; ++i) a.p[i] = c->p[i];
    for (int i = 0; i < 4; ++i) {
        a.in[i] = c->s64[from][i];
        a.out[i] = c->s64[1 - from][i];
    }
    a.layer = c->layer;
    a.norm = c->norm;
    a.fail_key = c->d_key;
    a.own0 = c->own_c0;
    a.own1 = c->own_c1;
    a.coef = c->d_coef;
    a.wall_kind = c->d_wall_kind;
    a.star = StarTab{c->d_star, c->d_star ? c->d_star + 6 * c->cells() : nullptr, c->cells()};
    a.q_rad = c->has_rad ? c->d_qrad : nullptr;
    a.dom_key = c->d_dom;
    if (c->coeff_kind == HYG_COEFF_MATERIAL) a.coeff_kind = kCoeffMaterial;
    return a;
}

StarArgs star_args(hyg_ctx* c, const double* u, const double* v, bool strict, int64_t layer) {
    StarArgs s{};
    s.n_walls = c->n_walls;
    s.n = c->n;
    s.u = u;
    s.v = v;
    s.wall_kind = c->d_wall_kind;
    for (int i = 0; i < 4; ++i) s.p[i] = c->p[i];
    s.T_i = c->T_i;
    s.P_vi = c->P_vi;
    s.ref = c->d_ref;
    s.strict = strict ? 1 : 0;
    s.node = c->d_star;
    s.half = c->d_star + 6 * c->cells();
    s.cells = c->cells();
    s.layer = layer;
    s.fail_key = c->d_key;
    s.dom_key = c->d_dom;
    s.own0 = c->own_c0;
    s.own1 = c->own_c1;
    s.exact = c->mat_exact ? 1 : 0;
    return s;
}

// StarTables of layer (u, v) for every nonlinear wall into c->d_star.
int launch_star_tables(hyg_ctx* c, const double* u, const double* v, bool strict, int64_t layer,
                       hyg_status* status) {
    if (!c->d_star) HYG_CUDA(cudaMalloc(&c->d_star, sizeof(double) * 9 * static_cast<size_t>(c->cells())));
    StarArgs s = star_args(c, u, v, strict, layer);
    LaunchScope ls(c, strict ? "star_tables" : "star_tables_clamped", static_cast<double>(c->cells()));
    k_star_tables<<<static_cast<int>((c->cells() + 127) / 128), 128, 0, c->stream>>>(s);
    return HYG_OK;
}

// radiation_fluxes (building.cpp:88-105) from the wall temperature layer u into c->d_qrad
void launch_radiation(hyg_ctx* c, const double* u) {
    RadArgs r{};
    r.n_targets = 2 * c->n_walls;
    r.tgt_off = c->d_rad_tgt;
    r.grp_off = c->d_rad_grp;
    r.grp_num = c->d_rad_num;
    r.grp_den = c->d_rad_den;
    r.t_e = c->d_rad_e;
    r.t_r = c->d_rad_r;
    r.t_coef = c->d_rad_coef;
    r.T_i = c->T_i;
    r.u = u;
    r.q = c->d_qrad;
    LaunchScope ls(c, "radiation", 0.0);
    k_radiation<<<(r.n_targets + 127) / 128, 128, 0, c->stream>>>(r);
}

// a strict evaluation left the material box in the step into layer `lay`
int domain_failure(hyg_ctx* c, int64_t lay, hyg_status* st) {
    unsigned long long dom = ~0ull;
    cudaMemcpy(&dom, c->d_dom, sizeof dom, cudaMemcpyDeviceToHost);
    const int w = static_cast<int>(dom >> 32);
    const unsigned order = static_cast<unsigned>(dom & 0xffffffffu);
    const bool half = order >= static_cast<unsigned>(c->n);
    const int j = static_cast<int>(half ? order - c->n : order);
    if (st) {
        st->code = HYG_EDOMAIN;
        st->layer = lay;
        st->wall = w;
        st->node = j;
        st->half = half ? 1 : 0;
        st->t_star = c->t;
        if (half)
            std::snprintf(st->message, sizeof st->message,
                          "material state outside admissible box in wall %d [half node %d+1/2] (step into layer %lld)",
                          w, j, static_cast<long long>(lay));
        else
            std::snprintf(st->message, sizeof st->message,
                          "material state outside admissible box in wall %d [node %d] (step into layer %lld)", w, j,
                          static_cast<long long>(lay));
    }
    return HYG_EDOMAIN;
}

int read_key(hyg_ctx* c, unsigned long long* key, hyg_status* status) {
    HYG_CUDA(cudaMemcpyAsync(key, c->d_key, sizeof *key, cudaMemcpyDeviceToHost, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int diverged(hyg_ctx* c, unsigned long long key, hyg_status* st) {
    const int64_t lay = static_cast<int64_t>(key >> 32);
    const unsigned w = static_cast<unsigned>(key & 0xffffffffu);
    if (st) {
        st->code = HYG_EDIVERGED;
        st->layer = lay;
        st->wall = w == 0xffffffffu ? -1 : static_cast<int>(w);
        st->t_star = c->t;
        if (w == 0xffffffffu) {
            std::snprintf(st->message, sizeof st->message, "zone state diverged at t* = %.17g", c->t);
        } else {
            std::snprintf(st->message, sizeof st->message,
                          "field norm exceeded %.17g in wall %u at t* = %.17g (layer %lld)", c->norm, w,
                          c->t, static_cast<long long>(lay));
        }
    }
    return HYG_EDIVERGED;
}

// ---- the per-step path ---------------------------------------------------------
// After a one-step kernel wrote the new layer into s64[1-cur][1] / [3]:
// u_prev <- u_curr, u_curr <- new, and the old u_prev buffer becomes the
// scratch slot (pointer rotation of wall.cpp:80-83, no copies).
void rotate_layers(hyg_ctx* c) {
    double** s = c->s64[c->cur];
    double** t = c->s64[1 - c->cur];
    for (int f = 0; f < 4; f += 2) {       // f = 0: u, f = 2: v
        double* old_prev = s[f];
        s[f] = s[f + 1];
        s[f + 1] = t[f + 1];
        t[f + 1] = old_prev;
    }
}

int advance_general(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status) {
    if (c->precision != HYG_F64) {
        set_status(status, HYG_ENOTSUP, "fp32 state needs a fused grid (N in {64,128,256,512})");
        return HYG_ENOTSUP;
    }
    const int64_t block = 65536;     // forcing rows per upload
    if (c->coeff_kind != HYG_COEFF_ANALYTIC_D && c->coef_dt != dt) {
        LaunchScope ls(c, "coupled_coef", 0.0);
        k_coupled_coef<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(c->n_walls, c->dx, dt, c->d_groups,
                                                                         c->d_biot, c->d_coef);
        c->coef_dt = dt;
    }
    const int kind = c->coeff_kind == HYG_COEFF_MATERIAL ? kCoeffMaterial
                     : c->coeff_kind == HYG_COEFF_ANALYTIC_D ? kCoeffAnalyticD
                                                             : kCoeffConstant;
    HYG_CUDA(cudaMemsetAsync(c->d_key, 0xff, sizeof(unsigned long long), c->stream));
    HYG_CUDA(cudaMemsetAsync(c->d_dom, 0xff, sizeof(unsigned long long), c->stream));
    for (int64_t done = 0; done < nsteps;) {
        const int64_t rows = std::min(block, nsteps - done);
        std::vector<double> times(rows);
        double t = c->t;
        for (int64_t k = 0; k < rows; ++k) {
            times[k] = t;
            t += dt;
        }
        int rc = upload_table(c, c->layer, times, status);
        if (rc) return rc;
        if (!c->zones.empty()) {
            rc = upload_src(c, c->layer, times, status);
            if (rc) return rc;
        }
        const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
        const int threads = 256;
        const int cells_per_block = step_cells(kind);
        const int grid = static_cast<int>((c->cells() + cells_per_block - 1) / cells_per_block);
        const int nsrc = static_cast<int>(c->zsrc.size() / 3);
        double* ptr0[2][4];
        std::memcpy(ptr0, c->s64, sizeof ptr0);
        for (int64_t k = 0; k < rows; ++k) {
            // layer-n radiation fluxes and frozen coefficients (building.cpp:158; wall.cpp:206)
            if (c->has_rad) launch_radiation(c, c->s64[c->cur][1]);
            StepArgs a = step_args(c, c->cur, dt);
            a.amb = c->d_table + k * nch;
            a.layer = c->layer + k;
            if (kind == kCoeffMaterial) {
                // StarTables + rows + zones in one launch (k_material_step)
                const StarArgs sa = star_args(c, a.in[1], a.in[3], true, c->layer + k);
                ZoneArgs z{};
                if (!c->zones.empty()) {
                    z.n_zones = static_cast<int>(c->zones.size());
                    z.n = c->n;
                    z.dt = dt;
                    z.zones = c->d_zones;
                    z.links = c->d_zlinks;
                    z.inz = c->d_inz;
                    z.src = c->d_src + k * (nsrc * 3 + 2);
                    z.n_sources = nsrc;
                    z.uc = c->s64[c->cur][1];
                    z.vc = c->s64[c->cur][3];
                    z.zu_in = c->zu[c->zcur];
                    z.zv_in = c->zv[c->zcur];
                    z.zu_out = c->zu[1 - c->zcur];
                    z.zv_out = c->zv[1 - c->zcur];
                    z.layer = c->layer + k;
                    z.norm = c->norm;
                    z.fail_key = c->d_key;
                    z.own0 = c->own_z0;
                    z.own1 = c->own_z1;
                }
                const int mgrid = static_cast<int>((c->cells() + kMatCells - 1) / kMatCells);
                const int zblocks = (z.n_zones + kMatThreads - 1) / kMatThreads;
                LaunchScope ls(c, "material_step", static_cast<double>(c->cells()));
                if (c->mat_exact) k_material_step<true><<<mgrid + zblocks, kMatThreads, 0, c->stream>>>(a, sa, z, mgrid);
                else k_material_step<false><<<mgrid + zblocks, kMatThreads, 0, c->stream>>>(a, sa, z, mgrid);
                if (!c->zones.empty()) c->zcur ^= 1;
            } else if (c->zones.empty()) {
                LaunchScope ls(c, "df_step_general", static_cast<double>(c->cells()));
                if (kind == kCoeffConstant)
                    k_df_step_general<kCoeffConstant><<<grid, threads, 0, c->stream>>>(a);
                else
                    k_df_step_general<kCoeffAnalyticD><<<grid, threads, 0, c->stream>>>(a);
            } else {
                ZoneArgs z{};
                z.n_zones = static_cast<int>(c->zones.size());
                z.n = c->n;
                z.dt = dt;
                z.zones = c->d_zones;
                z.links = c->d_zlinks;
                z.inz = c->d_inz;
                z.src = c->d_src + k * (nsrc * 3 + 2);
                z.n_sources = nsrc;
                z.uc = c->s64[c->cur][1];    // layer n samples (building.cpp:162-164)
                z.vc = c->s64[c->cur][3];
                z.zu_in = c->zu[c->zcur];
                z.zv_in = c->zv[c->zcur];
                z.zu_out = c->zu[1 - c->zcur];
                z.zv_out = c->zv[1 - c->zcur];
                z.layer = c->layer + k;
                z.norm = c->norm;
                z.fail_key = c->d_key;
                z.own0 = c->own_z0;
                z.own1 = c->own_z1;
                const int zblocks = (z.n_zones + threads - 1) / threads;
                LaunchScope ls(c, "building_step", static_cast<double>(c->cells()));
                if (kind == kCoeffConstant)
                    k_building_step<kCoeffConstant><<<grid + zblocks, threads, 0, c->stream>>>(a, z, grid);
                else
                    k_building_step<kCoeffAnalyticD><<<grid + zblocks, threads, 0, c->stream>>>(a, z, grid);
                c->zcur ^= 1;
            }
            rotate_layers(c);
        }
        HYG_CUDA(cudaGetLastError());
        unsigned long long key;
        rc = read_key(c, &key, status);
        if (rc) return rc;
        if (key != ~0ull) {
            // kernels after the failing step returned early: replay only the
            // rotations of the steps that ran
            const int64_t fail_layer = static_cast<int64_t>(key >> 32);
            unsigned long long dom = ~0ull;
            if (c->any_material)
                HYG_CUDA(cudaMemcpy(&dom, c->d_dom, sizeof dom, cudaMemcpyDeviceToHost));
            // divergence: the failing layer exists; domain error: its step never ran
            const int64_t ran = fail_layer - c->layer - (dom != ~0ull ? 1 : 0);
            std::memcpy(c->s64, ptr0, sizeof ptr0);
            for (int64_t k = 0; k < ran; ++k) rotate_layers(c);
            if (!c->zones.empty() && (rows - ran) % 2) c->zcur ^= 1;
            c->t = ran < rows ? times[ran] : t;
            c->layer += ran;
            if (dom != ~0ull) return domain_failure(c, fail_layer, status);
            return diverged(c, key, status);
        }
        c->t = t;
        c->layer += rows;
        done += rows;
    }
    return HYG_OK;
}

// ---- the fused path (K1) -----------------------------------------------------------
template <typename Real>
int advance_fused_t(hyg_ctx* c, Real* (&buf)[2][4], int64_t nsteps, double dt, hyg_status* status) {
    if (c->coef_dt != dt) {
        LaunchScope ls(c, "coupled_coef", 0.0);
        k_coupled_coef<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(c->n_walls, c->dx, dt, c->d_groups,
                                                                         c->d_biot, c->d_coef);
        c->coef_dt = dt;
    }
    int lpw = 16;
    SegFn<Real> fast = pick_seg<Real>(c->n, c->flux, false, &lpw);
    SegFn<Real> exact = pick_seg<Real>(c->n, c->flux, true, &lpw);
    const int walls_per_cta = kWarps * 32 / lpw;
    const int grid = (c->n_walls + walls_per_cta - 1) / walls_per_cta;
    const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
    const int smem = kChunk * nch * static_cast<int>(sizeof(Ambient));
    if (smem > 64 * 1024) {
        set_status(status, HYG_ENOTSUP, "too many forcing channels for the fused kernel");
        return HYG_ENOTSUP;
    }
    const int64_t block = 1 << 18;    // layers per table upload
    for (int64_t done = 0; done < nsteps;) {
        const int64_t rows = std::min(block, nsteps - done);
        std::vector<double> times(rows);
        double t = c->t;
        for (int64_t k = 0; k < rows; ++k) {
            times[k] = t;
            t += dt;
        }
        int rc = upload_table(c, c->layer, times, status);
        if (rc) return rc;
        HYG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        HYG_CUDA(cudaMemsetAsync(c->d_key, 0xff, sizeof(unsigned long long), c->stream));
        CoupledSegArgs<Real> a{};
        a.n_walls = c->n_walls;
        a.n_channels = nch;
        a.divergence_norm = c->norm;
        a.coef = c->d_coef;
        a.chan = c->d_chan;
        a.stop = c->d_flag;
        a.suspect = c->d_flag;
        a.fail_key = c->d_key;
        const int cur0 = c->cur;
        // the bit-30 test proves |x| <= norm only for norm >= 2 (fp32 deviations: 3);
        // below that every segment runs the exact guard
        const bool fast_ok = c->norm >= (sizeof(Real) == 4 ? 3.0 : 2.0);
        int nseg = 0;
        for (int64_t s0 = 0; s0 < rows; s0 += c->seg_len, ++nseg) {
            if (!fast_ok) continue;
            const int len = static_cast<int>(std::min<int64_t>(c->seg_len, rows - s0));
            a.nsteps = len;
            a.layer0 = c->layer + s0;
            a.table = c->d_table + s0 * nch;
            a.seg_index = nseg;
            const int from = (cur0 + nseg) & 1;
            for (int i = 0; i < 4; ++i) {
                a.in[i] = buf[from][i];
                a.out[i] = buf[1 - from][i];
            }
            LaunchScope ls(c, sizeof(Real) == 8 ? "df_coupled_fused_f64" : "df_coupled_fused_f32",
                           static_cast<double>(c->cells()) * len);
            fast(a, grid, smem, c->stream, c->device);
        }
        HYG_CUDA(cudaGetLastError());
        int flag = 0;
        HYG_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
        HYG_CUDA(cudaStreamSynchronize(c->stream));
        if (!fast_ok) flag = 1;           // exact guard from the first segment
        if (flag == 0) {
            c->cur = (cur0 + nseg) & 1;
            c->t = t;
            c->layer += rows;
            done += rows;
            continue;
        }
        // The fast guard fired: flag = index + 1 of the first flagged segment K.
        // Later segments returned without writing, so buf[(cur0 + K) & 1] still
        // holds K's input.  Replay K.. with the exact per-step guard of
        // check_bounded (building.cpp:282-300); stop at the first failure.
        const int K = flag - 1;
        auto time_of = [&](int64_t L) {   // time of absolute layer L inside this block
            const int64_t i = L - c->layer;
            return i < rows ? times[i] : t;
        };
        for (int k = K; k < nseg; ++k) {
            const int from = (cur0 + k) & 1;
            const int64_t s0 = static_cast<int64_t>(k) * c->seg_len;
            const int len = static_cast<int>(std::min<int64_t>(c->seg_len, rows - s0));
            a.nsteps = len;
            a.layer0 = c->layer + s0;
            a.seg_index = k;
            a.table = c->d_table + s0 * nch;
            for (int i = 0; i < 4; ++i) {
                a.in[i] = buf[from][i];
                a.out[i] = buf[1 - from][i];
            }
            HYG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
            {
                LaunchScope ls(c, sizeof(Real) == 8 ? "df_coupled_exact_f64" : "df_coupled_exact_f32",
                               static_cast<double>(c->cells()) * len);
                exact(a, grid, smem, c->stream, c->device);
            }
            HYG_CUDA(cudaGetLastError());
            unsigned long long key;
            rc = read_key(c, &key, status);
            if (rc) return rc;
            if (key != ~0ull) {
                // walls that failed stopped at their failing layer (curr = the
                // failing layer), the others at the segment end; the state is a
                // diagnostic snapshot, `layer` names the first failing layer
                c->cur = 1 - from;
                const int64_t L = static_cast<int64_t>(key >> 32);
                c->t = time_of(L);
                c->layer = L;
                return diverged(c, key, status);
            }
        }
        // |x| >= 2 somewhere but within the norm: the exact replay produced the
        // same state the fast pass would have
        c->cur = (cur0 + nseg) & 1;
        c->t = t;
        c->layer += rows;
        done += rows;
    }
    return HYG_OK;
}

// ---- the fused nonlinear path (K2w, analytic d(v), one warp per wall) -------------
constexpr int kSplitWallsMax = 148;   // one CTA per SM at most

template <int NPT, int M>
void launch_dv_walls_m(const NonlinearSegArgs& a, int m, cudaStream_t s) {
    if constexpr (M <= NPT) {
        if (m != M) return launch_dv_walls_m<NPT, M + 1>(a, m, s);
        const int grid = (a.n_walls + kDvWarps - 1) / kDvWarps;
        k_dv_walls<NPT, M><<<grid, kDvWarps * 32, 0, s>>>(a);
    }
}

template <int NW>
void launch_dv_split(const NonlinearSegArgs& a, int nw, cudaStream_t s) {
    if constexpr (NW <= 8) {
        if (nw != NW) return launch_dv_split<NW + 1>(a, nw, s);
        k_dv_wall_split<NW><<<a.n_walls, NW * 32, 0, s>>>(a);
    }
}

template <int NW, int H>
void launch_dv_halo(const NonlinearSegArgs& a, int nw, cudaStream_t s) {
    if constexpr (NW <= 8) {
        if (nw != NW) return launch_dv_halo<NW + 1, H>(a, nw, s);
        k_dv_wall_halo<NW, H><<<a.n_walls, NW * 32, 0, s>>>(a);
    }
}

// n <= 256.  Fewer walls than SMs: K2h/K2s (a wall over ceil(n/32) warps, latency).
// Otherwise K2w: NPT = the smallest power of two with 32 NPT >= n, M = nodes of
// the reversed lane.
void launch_dv_walls(const NonlinearSegArgs& a, int n, cudaStream_t s) {
    if (a.n_walls <= kSplitWallsMax && n > 32) {
        // K2h when the same ceil(n/32) warps leave H >= 2 halo lanes a side
        // (configs[0]: n = 101, 4 warps, H = 3: a barrier every 3 steps)
        const int nw = (n + 31) / 32, halo = std::min(6, (32 - (n + nw - 1) / nw) / 2);
        switch (halo) {
            case 2: return launch_dv_halo<1, 2>(a, nw, s);
            case 3: return launch_dv_halo<1, 3>(a, nw, s);
            case 4: return launch_dv_halo<1, 4>(a, nw, s);
            case 5: return launch_dv_halo<1, 5>(a, nw, s);
            case 6: return launch_dv_halo<1, 6>(a, nw, s);
            default: break;
        }
    }
    if (a.n_walls <= kSplitWallsMax && n >= 3) return launch_dv_split<1>(a, (n + 31) / 32, s);
    const int npt = n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
    const int m = n - (n - 1) / npt * npt;
    switch (npt) {
        case 1: launch_dv_walls_m<1, 1>(a, m, s); break;
        case 2: launch_dv_walls_m<2, 1>(a, m, s); break;
        case 4: launch_dv_walls_m<4, 1>(a, m, s); break;
        default: launch_dv_walls_m<8, 1>(a, m, s); break;
    }
}

int advance_nonlinear(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status) {
    // the fused kernels carry the fast guard only: it proves |x| <= norm for norm >= 2
    if (!(c->norm >= 2.0)) return advance_general(c, nsteps, dt, status);
    const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
    const int64_t block = 1 << 18;
    for (int64_t done = 0; done < nsteps;) {
        const int64_t rows = std::min(block, nsteps - done);
        std::vector<double> times(rows);
        double t = c->t;
        for (int64_t k = 0; k < rows; ++k) {
            times[k] = t;
            t += dt;
        }
        int rc = upload_table(c, c->layer, times, status);
        if (rc) return rc;
        HYG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        NonlinearSegArgs a{};
        a.n_walls = c->n_walls;
        a.n = c->n;
        a.n_channels = nch;
        a.dx = c->dx;
        a.dt = dt;
        for (int i = 0; i < 4; ++i) a.p[i] = c->p[i];
        a.groups = c->d_groups;
        a.biot = c->d_biot;
        a.chan = c->d_chan;
        a.stop = c->d_flag;
        a.suspect = c->d_flag;
        const int cur0 = c->cur;
        int nseg = 0;
        for (int64_t s0 = 0; s0 < rows; s0 += c->seg_len, ++nseg) {
            const int len = static_cast<int>(std::min<int64_t>(c->seg_len, rows - s0));
            a.nsteps = len;
            a.layer0 = c->layer + s0;
            a.seg_index = nseg;
            a.table = c->d_table + s0 * nch;
            const int from = (cur0 + nseg) & 1;
            for (int i = 0; i < 4; ++i) {
                a.in[i] = c->s64[from][i];
                a.out[i] = c->s64[1 - from][i];
            }
            LaunchScope ls(c, "df_analytic_fused", static_cast<double>(c->cells()) * len);
            if (c->n <= 32 * 8) launch_dv_walls(a, c->n, c->stream);
            else k_df_analytic_walls<1024, 256><<<c->n_walls, 288, 0, c->stream>>>(a);
        }
        HYG_CUDA(cudaGetLastError());
        int flag = 0;
        HYG_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
        HYG_CUDA(cudaStreamSynchronize(c->stream));
        if (flag == 0) {
            c->cur = (cur0 + nseg) & 1;
            c->t = t;
            c->layer += rows;
            done += rows;
            continue;
        }
        // the fast guard fired in segment K (whose input is intact): march the
        // rest of the request with the per-step kernel and its exact guard
        const int64_t k0 = static_cast<int64_t>(flag - 1) * c->seg_len;
        c->cur = (cur0 + flag - 1) & 1;
        c->t = times[k0];
        c->layer += k0;
        return advance_general(c, nsteps - done - k0, dt, status);
    }
    return HYG_OK;
}

// ---- the temporally blocked long-wall path (K3, analytic d(v), one wall) ----------
constexpr int kTileNPT = 8;             // K3w: W = 256-node windows, S = 8 steps per launch
constexpr int kTileS = kTileNPT;

int advance_tiled(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status) {
    if (!(c->norm >= 2.0)) return advance_general(c, nsteps, dt, status);   // fast guard: norm >= 2 only
    const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
    const int64_t block = 1 << 18;
    for (int64_t done = 0; done < nsteps;) {
        const int64_t rows = std::min(block, nsteps - done);
        std::vector<double> times(rows);
        double t = c->t;
        for (int64_t k = 0; k < rows; ++k) {
            times[k] = t;
            t += dt;
        }
        int rc = upload_table(c, c->layer, times, status);
        if (rc) return rc;
        HYG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        TiledArgs a{};
        a.n = c->n;
        a.n_channels = nch;
        a.chl = c->attach[0].index;
        a.chr = c->attach[1].index;
        a.dx = c->dx;
        a.dt = dt;
        for (int i = 0; i < 4; ++i) a.p[i] = c->p[i];
        a.groups = c->groups[0];
        a.bl = c->biot[0];
        a.br = c->biot[1];
        a.stop = c->d_flag;
        a.suspect = c->d_flag;
        using G = DvTiles<kTileNPT>;
        const int64_t tr = G::rface(c->n);
        // persistent interior kernel: as many CTAs as fit at once (each warp
        // walks the windows with a stride of all warps), 16-byte stores need
        // 16-byte aligned windows: T and NPT even, the buffers 256-byte aligned
        const bool tma = c->tmaps_ok && c->tiled_load == 0;
        int per_sm = 1;
        if (tma) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dv_tiled_tma<kTileNPT, kK3MinB>, kDvWarps * 32, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dv_tiled_stream<kTileNPT, kK3MinB>, kDvWarps * 32, 0);
        per_sm = std::max(per_sm, 1);
        const int n_sm = sm_count(c->device);
        const int grid = static_cast<int>(std::min<int64_t>((tr - 1 + kDvWarps - 1) / kDvWarps,
                                                            static_cast<int64_t>(per_sm) * n_sm));
        // cells owned by the face windows (window 0 and t >= tr) and by the interior ones
        const double face_cells = static_cast<double>(G::W - kTileNPT) + static_cast<double>(c->n - (tr * G::T + kTileNPT));
        const double mid_cells = static_cast<double>(c->cells()) - face_cells;
        const int cur0 = c->cur;
        int nseg = 0;
        for (int64_t s0 = 0; s0 < rows; s0 += kTileS, ++nseg) {
            a.steps = static_cast<int>(std::min<int64_t>(kTileS, rows - s0));
            a.seg_index = nseg;
            a.table = c->d_table + s0 * nch;
            const int from = (cur0 + nseg) & 1;
            for (int i = 0; i < 4; ++i) {
                a.in[i] = c->s64[from][i];
                a.out[i] = c->s64[1 - from][i];
            }
            auto interior = [&](int64_t t0, int64_t t1) {
                if (t1 <= t0) return;
                TiledArgs ai = a;
                ai.t_begin = t0;
                ai.t_end = t1;
                const int g = static_cast<int>(std::min<int64_t>((t1 - t0 + kDvWarps - 1) / kDvWarps, std::max(grid, 1)));
                if (tma) k_dv_tiled_tma<kTileNPT, kK3MinB><<<g, kDvWarps * 32, 0, c->stream>>>(ai, c->tmaps[from]);
                else k_dv_tiled_stream<kTileNPT, kK3MinB><<<g, kDvWarps * 32, 0, c->stream>>>(ai);
            };
            {
                LaunchScope ls(c, "df_analytic_tiled", mid_cells * a.steps);
                if (c->ov_event) {
                    // overlapped halo refresh (hyg_advance_overlapped): window t reads cells
                    // [t T, t T + W); those clear of the refreshed cells march while the
                    // exchange is still in flight, the rest behind its event
                    const int64_t t_lo = std::min<int64_t>(tr, std::max<int64_t>(1, (c->ov_lo + G::T - 1) / G::T));
                    const int64_t t_hi = std::max<int64_t>(
                        t_lo, std::min<int64_t>(tr, c->ov_hi > 0 ? (c->n - c->ov_hi - G::W) / G::T + 1 : tr));
                    interior(t_lo, t_hi);
                    HYG_CUDA(cudaStreamWaitEvent(c->stream, c->ov_event, 0));
                    interior(1, t_lo);
                    interior(t_hi, tr);
                    c->ov_event = nullptr;
                } else {
                    interior(1, tr);
                }
            }
            LaunchScope ls(c, "df_analytic_tiled_faces", face_cells * a.steps);
            k_dv_tiled<kTileNPT, true><<<1, kDvWarps * 32, 0, c->stream>>>(a);
        }
        HYG_CUDA(cudaGetLastError());
        int flag = 0;
        HYG_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
        HYG_CUDA(cudaStreamSynchronize(c->stream));
        if (flag == 0) {
            c->cur = (cur0 + nseg) & 1;
            c->t = t;
            c->layer += rows;
            done += rows;
            continue;
        }
        // fast guard fired in launch K (input intact): exact per-step path from there
        const int64_t k0 = static_cast<int64_t>(flag - 1) * kTileS;
        c->cur = (cur0 + flag - 1) & 1;
        c->t = times[k0];
        c->layer += k0;
        return advance_general(c, nsteps - done - k0, dt, status);
    }
    return HYG_OK;
}

// ---- the zone-ring temporally blocked path (K4, K4r) -----------------------------
// grid_cap > 0 (HYG_TUNE_RING_GRID) bounds the persistent grid, so each CTA
// walks several zone blocks (the next-block prefetch path) even in small rings
template <int NPT>
void launch_ring_reg(const RingArgs& a, int threads, size_t smem, cudaStream_t s, int device, bool small,
                     int grid_cap) {
    // small: every zone has <= 6 wall links and <= 2 ring peers (configs[3])
    auto k = small ? k_ring_reg<NPT, kRingRegS, 6, 2> : k_ring_reg<NPT, kRingRegS>;
    ensure_smem_attr(k, device, 227 * 1024);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    const int nblk = (a.n_zones + a.B - 1) / a.B;
    int grid = std::max(1, std::min(nblk, std::max(per_sm, 1) * sm_count(device)));
    if (grid_cap > 0) grid = std::min(grid, grid_cap);
    k<<<grid, threads, smem, s>>>(a);
}

void launch_ring_pipe(const RingArgs& a, size_t smem, cudaStream_t s, int device, int grid_cap) {
    using Sh = RingPipeShape<kRingPipeS>;
    auto k = k_ring_pipe<kRingPipeS, Sh::kThreads>;
    ensure_smem_attr(k, device, 227 * 1024);
    const int nblk = (a.n_zones + a.B - 1) / a.B;
    int grid = std::max(1, std::min(nblk, sm_count(device)));
    if (grid_cap > 0) grid = std::min(grid, grid_cap);
    k<<<grid, Sh::threads(a.B, a.W), smem, s>>>(a);
}

// K6 (k_ring_split.cuh): phase 1 (zone air + wall cones, records the air series),
// then phase 2 (every wall in registers, no barrier per step)
void launch_ring_cone(const RingArgs& a, double* series, int LB, bool small, cudaStream_t s, int device,
                      const double* rowsT, const double* zpT, const ConeIO& io) {
    using Sh = RingConeShape<kRingSplitS>;
    auto k = small ? k_ring_cone<kRingSplitS, 6, 2> : k_ring_cone<kRingSplitS>;
    const int rw = RingShape<8, kRingSplitS>::row_width(a.n_channels, a.n_sources);
    const size_t smem = Sh::smem_doubles(LB, a.W, rw) * sizeof(double);
    ensure_smem_attr(k, device, 227 * 1024);
    const int OB = LB - 2 * kRingSplitS;
    k<<<(a.n_zones + OB - 1) / OB, Sh::threads(LB, a.W), smem, s>>>(a, series, LB, rowsT, zpT, io);
}

// tails of depth DIN (state arrays or a previous stub's output) -> tails of depth DIN - S, S steps later
template <int DIN>
void launch_ring_stub(const RingArgs& a, const double* series, const double* rowsT, const ConeIO& in,
                      double* const (&out)[4], cudaStream_t s, int /*device*/) {
    const int walls = a.n_zones * a.W;
    k_ring_stub<DIN, kRingSplitS><<<(walls + 127) / 128, 128, 0, s>>>(a, series, rowsT, in, out[0], out[1], out[2], out[3]);
}

template <int NPT, int SW, bool TMAP>
void launch_ring_walls_sw(const RingArgs& a, const double* series, cudaStream_t s, int device, int grid_cap,
                          const TiledMaps& mi, const TiledMaps& mo) {
    auto k = k_ring_walls<NPT, SW, TMAP>;
    const size_t smem = RingWallShape<NPT>::smem_doubles(SW, a.n_channels, kRingWallWarps) * sizeof(double) +
                        (TMAP ? 1024 : 0);
    ensure_smem_attr(k, device, 100 * 1024);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * kRingWallWarps, smem);
    const int pairs = (a.n_zones * a.W + 1) / 2, nblk = (pairs + kRingWallWarps - 1) / kRingWallWarps;
    int grid = std::max(1, std::min(nblk, std::max(per_sm, 1) * sm_count(device)));
    if (grid_cap > 0) grid = std::min(grid, grid_cap);   // HYG_TUNE_RING_GRID: several pairs per warp in small rings
    k<<<grid, 32 * kRingWallWarps, smem, s>>>(a, series, mi, mo);
}

// m: cone launches per walls launch (the series row of a zone has m S slots); maps: the
// state arrays' tensor maps (n = 128 and an even wall count), else the 1-D bulk copies
template <int NPT>
void launch_ring_walls(const RingArgs& a, const double* series, cudaStream_t s, int device, int grid_cap, int m,
                       const TiledMaps* mi, const TiledMaps* mo) {
    static const TiledMaps none{};
    if constexpr (NPT == 8) {
        if (mi && mo) {
            if (m == 1) launch_ring_walls_sw<8, kRingSplitS, true>(a, series, s, device, grid_cap, *mi, *mo);
            else if (m == 2) launch_ring_walls_sw<8, 2 * kRingSplitS, true>(a, series, s, device, grid_cap, *mi, *mo);
            else launch_ring_walls_sw<8, 3 * kRingSplitS, true>(a, series, s, device, grid_cap, *mi, *mo);
            return;
        }
    }
    if (m == 1) launch_ring_walls_sw<NPT, kRingSplitS, false>(a, series, s, device, grid_cap, none, none);
    else if (m == 2) launch_ring_walls_sw<NPT, 2 * kRingSplitS, false>(a, series, s, device, grid_cap, none, none);
    else launch_ring_walls_sw<NPT, 3 * kRingSplitS, false>(a, series, s, device, grid_cap, none, none);
}

template <int NPT>
void launch_ring(const RingArgs& a, int grid, int threads, size_t smem, cudaStream_t s, int device) {
    auto k = k_ring_tiled<NPT, kRingS>;
    ensure_smem_attr(k, device, 227 * 1024);
    k<<<grid, threads, smem, s>>>(a);
}

int advance_ring(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status, bool reg = true) {
    // K4r by default; K5 (pipelined, S = 12, HYG_TUNE_RING_KERNEL = 3) measured slower
    // (2.8e11 vs 3.4e11: the per-step critical path binds, not HBM)
    const int rk = c->ring_kernel == 0 ? kRingAuto : c->ring_kernel;
    const bool pipe = reg && c->ring_pipe_B > 0 && c->norm >= 2.0 && rk == 3;
    // K6: the split march (no per-step barrier on the walls' path), the default
    const bool split = reg && c->ring_cone_LB > 0 && c->norm >= 2.0 && rk == 4;
    if (rk == 2) reg = false;
    if (c->coef_dt != dt) {
        LaunchScope ls(c, "coupled_coef", 0.0);
        k_coupled_coef<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(c->n_walls, c->dx, dt, c->d_groups,
                                                                         c->d_biot, c->d_coef);
        c->coef_dt = dt;
    }
    if (split && c->rows_dt != dt) {
        LaunchScope ls(c, "ring_cone_rows", 0.0);
        k_ring_cone_rows<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(c->n_walls, c->d_coef, c->d_ring_rowsT);
        c->rows_dt = dt;
    }
    const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
    const int nsrc = static_cast<int>(c->zsrc.size() / 3);
    // K4r needs the fast guard (norm >= 2: a clear bit 30 proves |x| < 2); a
    // flagged K4r launch is replayed by K4 and its exact guard
    reg = reg && c->ring_reg_B > 0 && c->norm >= 2.0;
    const int Z = static_cast<int>(c->zones.size()), W = c->ring_W, npt = c->n / 16;
    const int B = pipe ? c->ring_pipe_B : reg ? c->ring_reg_B : c->ring_B;
    const int grid = (Z + B - 1) / B;
    const int rw = RingShape<8, kRingS>::row_width(nch, nsrc);
    const int split_m = std::min(std::max(c->ring_split_m, 1), kRingSplitMaxM);
    const int S = split ? split_m * kRingSplitS : pipe ? kRingPipeS : reg ? kRingRegS : kRingS;   // steps per launch
    const int threads = reg ? RingRegShape<8, kRingRegS>::threads(B, W) : RingShape<8, kRingS>::threads(B, W);
    const size_t smem = pipe ? RingPipeShape<kRingPipeS>::smem_doubles(B, W, rw) * sizeof(double)
                        : reg ? RingRegShape<8, kRingRegS>::smem_doubles(B, W, c->n, rw) * sizeof(double)
                        : npt == 4 ? RingShape<4, kRingS>::smem_bytes(B, W, nch, nsrc)
                        : npt == 8 ? RingShape<8, kRingS>::smem_bytes(B, W, nch, nsrc)
                                   : RingShape<16, kRingS>::smem_bytes(B, W, nch, nsrc);
    const int64_t block = 65536 / S * S;
    for (int64_t done = 0; done < nsteps;) {
        const int64_t rows = std::min(block, nsteps - done);
        std::vector<double> times(rows);
        double t = c->t;
        for (int64_t k = 0; k < rows; ++k) {
            times[k] = t;
            t += dt;
        }
        int rc = upload_table(c, c->layer, times, status);
        if (rc) return rc;
        rc = upload_src(c, c->layer, times, status);
        if (rc) return rc;
        HYG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        RingArgs a{};
        a.n_zones = Z;
        a.W = W;
        a.n = c->n;
        a.B = B;
        a.norm = c->norm;
        a.biot = c->d_biot;
        a.attach = c->d_attach;
        a.coef = c->d_coef;
        a.n_channels = nch;
        a.n_sources = nsrc;
        a.dt = dt;
        a.zones = c->d_zones;
        a.links = c->d_zlinks;
        a.inz = c->d_inz;
        a.zparams = c->d_ring_zp;
        a.stop = c->d_flag;
        a.dbg_skip = c->ring_dbg_skip;
        const int cur0 = c->cur, z0 = c->zcur;
        int nseg = 0;
        for (int64_t s0 = 0; s0 < rows; s0 += S, ++nseg) {
            a.steps = static_cast<int>(std::min<int64_t>(S, rows - s0));
            a.seg_index = nseg;
            a.table = c->d_table + s0 * nch;
            a.src = c->d_src + s0 * (3 * nsrc + 2);
            const int from = (cur0 + nseg) & 1, zf = (z0 + nseg) & 1;
            for (int i = 0; i < 4; ++i) {
                a.in[i] = c->s64[from][i];
                a.out[i] = c->s64[1 - from][i];
            }
            a.zu_in = c->zu[zf];
            a.zv_in = c->zv[zf];
            a.zu_out = c->zu[1 - zf];
            a.zv_out = c->zv[1 - zf];
            if (split) {
                // a.steps <= m S steps: one cone launch per S steps (the later ones on the
                // tails k_ring_stub marches from the launch's input), then the walls
                constexpr int CS = kRingSplitS, PS = RingConeShape<kRingSplitS>::kPS;
                const int steps = a.steps, nsub = (steps + CS - 1) / CS;
                ConeIO io{};
                io.ser_stride = S;
                for (int j = 0; j < nsub; ++j) {
                    if (j == 0) {
                        for (int i = 0; i < 4; ++i) io.tin[i] = a.in[i];
                        io.tstride = c->n;
                    } else {
                        // tails at the start of cone launch j: depth 9 + 8 (nsub - 1 - j), from depth + 8
                        ConeIO sin = io;                 // the previous launch's tails source and series slots
                        const int din = PS - 1 + CS * (nsub - j);   // depth at the start of launch j - 1
                        const int ds = (din + 1) & ~1;
                        sin.toff = j == 1 ? c->n - ds : 0;       // the state arrays' last ds nodes, else a whole tail row
                        LaunchScope ls(c, "ring_stub", 0.0);
                        if (din == PS - 1 + CS) launch_ring_stub<PS - 1 + CS>(a, c->d_ring_series, c->d_ring_rowsT, sin, c->d_ring_tail[j & 1], c->stream, c->device);
                        else launch_ring_stub<PS - 1 + 2 * CS>(a, c->d_ring_series, c->d_ring_rowsT, sin, c->d_ring_tail[j & 1], c->stream, c->device);
                        for (int i = 0; i < 4; ++i) io.tin[i] = c->d_ring_tail[j & 1][i];
                        io.tstride = (din - CS + 1) & ~1;
                    }
                    // this launch reads the last PS nodes of its tails
                    io.toff = io.tstride - PS;
                    io.ser_off = j * CS;
                    RingArgs ac = a;
                    ac.steps = std::min(CS, steps - j * CS);
                    ac.table = a.table + static_cast<size_t>(j) * CS * nch;
                    ac.src = a.src + static_cast<size_t>(j) * CS * (3 * nsrc + 2);
                    ac.zu_in = j == 0 ? a.zu_in : c->d_ring_zt[(j - 1) & 1][0];
                    ac.zv_in = j == 0 ? a.zv_in : c->d_ring_zt[(j - 1) & 1][1];
                    ac.zu_out = j == nsub - 1 ? a.zu_out : c->d_ring_zt[j & 1][0];
                    ac.zv_out = j == nsub - 1 ? a.zv_out : c->d_ring_zt[j & 1][1];
                    LaunchScope ls(c, "ring_cone", 0.0);
                    launch_ring_cone(ac, c->d_ring_series, c->ring_cone_LB, c->ring_reg_small, c->stream, c->device,
                                     c->d_ring_rowsT, c->d_ring_zpT, io);
                }
                LaunchScope ls(c, "ring_walls", static_cast<double>(c->cells()) * a.steps);
                const bool tmap = c->tmaps_ok && c->tiled_load == 0 && c->n_walls % 2 == 0;
                if (npt == 4) launch_ring_walls<4>(a, c->d_ring_series, c->stream, c->device, c->ring_grid_cap, split_m, nullptr, nullptr);
                else launch_ring_walls<8>(a, c->d_ring_series, c->stream, c->device, c->ring_grid_cap, split_m,
                                          tmap ? &c->tmaps[from] : nullptr, tmap ? &c->tmaps[1 - from] : nullptr);
                continue;
            }
            LaunchScope ls(c, pipe ? "ring_pipe" : reg ? "ring_reg" : "ring_tiled", static_cast<double>(c->cells()) * a.steps);
            if (pipe) {
                launch_ring_pipe(a, smem, c->stream, c->device, c->ring_grid_cap);
            } else if (reg) {
                if (npt == 4) launch_ring_reg<4>(a, threads, smem, c->stream, c->device, c->ring_reg_small, c->ring_grid_cap);
                else launch_ring_reg<8>(a, threads, smem, c->stream, c->device, c->ring_reg_small, c->ring_grid_cap);
            } else if (npt == 4) launch_ring<4>(a, grid, threads, smem, c->stream, c->device);
            else if (npt == 8) launch_ring<8>(a, grid, threads, smem, c->stream, c->device);
            else launch_ring<16>(a, grid, threads, smem, c->stream, c->device);
        }
        HYG_CUDA(cudaGetLastError());
        int flag = 0;
        HYG_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
        HYG_CUDA(cudaStreamSynchronize(c->stream));
        if (flag == 0) {
            c->cur = (cur0 + nseg) & 1;
            c->zcur = (z0 + nseg) & 1;
            c->t = t;
            c->layer += rows;
            done += rows;
            continue;
        }
        // the guard fired in launch K (its input intact): K4r -> K4 (exact guard)
        // from there, K4 -> the exact per-step path
        const int64_t k0 = static_cast<int64_t>(flag - 1) * S;
        c->cur = (cur0 + flag - 1) & 1;
        c->zcur = (z0 + flag - 1) & 1;
        c->t = times[k0];
        c->layer += k0;
        if (reg && !c->owned_partial) return advance_ring(c, nsteps - done - k0, dt, status, false);
        return advance_general(c, nsteps - done - k0, dt, status);
    }
    return HYG_OK;
}

int advance_fused(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status) {
    if (c->precision == HYG_F32) return advance_fused_t<float>(c, c->s32, nsteps, dt, status);
    return advance_fused_t<double>(c, c->s64, nsteps, dt, status);
}

int to_f32(hyg_ctx* c, hyg_status* status) {
    if (c->precision != HYG_F32) return HYG_OK;
    const int threads = 256;
    const int grid = static_cast<int>((c->cells() + threads - 1) / threads);
    for (int i = 0; i < 4; ++i) {
        LaunchScope ls(c, "to_dev32", 0.0);
        k_to_dev32<<<grid, threads, 0, c->stream>>>(c->cells(), c->s64[c->cur][i], c->s32[c->cur][i]);
    }
    HYG_CUDA(cudaGetLastError());
    return HYG_OK;
}

int from_f32(hyg_ctx* c, hyg_status* status) {
    if (c->precision != HYG_F32) return HYG_OK;
    const int threads = 256;
    const int grid = static_cast<int>((c->cells() + threads - 1) / threads);
    for (int i = 0; i < 4; ++i) {
        LaunchScope ls(c, "from_dev32", 0.0);
        k_from_dev32<<<grid, threads, 0, c->stream>>>(c->cells(), c->s32[c->cur][i], c->s64[c->cur][i]);
    }
    HYG_CUDA(cudaGetLastError());
    return HYG_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int hyg_abi_version(void) { return HYG_ABI_VERSION; }

const char* hyg_strerror(int code) {
    switch (code) {
        case HYG_OK: return "ok";
        case HYG_EINVAL: return "invalid argument";
        case HYG_ESCHEMA: return "schema error";
        case HYG_EDIVERGED: return "numerical error (divergence)";
        case HYG_EDOMAIN: return "domain error";
        case HYG_ECONVERGE: return "convergence error";
        case HYG_ESCALING: return "scaling error";
        case HYG_ECUDA: return "CUDA error";
        case HYG_ENOTSUP: return "not supported";
        default: return "unknown";
    }
}

int hyg_create(const hyg_model_desc* d, hyg_ctx** out, hyg_status* status) {
    clear_status(status);
    if (!d || !out) {
        set_status(status, HYG_EINVAL, "null argument");
        return HYG_EINVAL;
    }
    *out = nullptr;
    if (d->n_walls < 1 || d->n_nodes < 3 || !(d->dx > 0.0) || !d->groups || !d->biot || !d->attach) {
        set_status(status, HYG_EINVAL, "need n_walls >= 1, n_nodes >= 3 (Grid1D wall.cpp:14), dx > 0");
        return HYG_EINVAL;
    }
    if (!(d->dt > 0.0)) {   // BuildingModel::validate building.cpp:14
        set_status(status, HYG_ESCHEMA, "dt must be positive");
        return HYG_ESCHEMA;
    }
    if (d->coeff_kind != HYG_COEFF_CONSTANT && d->coeff_kind != HYG_COEFF_ANALYTIC_D &&
        d->coeff_kind != HYG_COEFF_MATERIAL) {
        set_status(status, HYG_ENOTSUP, "coefficient model not implemented on the device");
        return HYG_ENOTSUP;
    }
    if (d->coeff_kind == HYG_COEFF_MATERIAL) {
        bool need_ref = false;
        for (int w = 0; w < d->n_walls; ++w) {
            const int k = d->wall_coeff ? d->wall_coeff[w] : HYG_COEFF_MATERIAL;
            if (k != HYG_COEFF_CONSTANT && k != HYG_COEFF_MATERIAL) {
                set_status(status, HYG_EINVAL, "wall_coeff entries must be HYG_COEFF_CONSTANT or HYG_COEFF_MATERIAL");
                return HYG_EINVAL;
            }
            need_ref = need_ref || k == HYG_COEFF_MATERIAL;
        }
        if (need_ref && (!d->wall_reference || !(d->T_i > 0.0) || !(d->P_vi > 0.0))) {
            set_status(status, HYG_EINVAL, "material walls need wall_reference and a scaling context (T_i, P_vi > 0)");
            return HYG_EINVAL;
        }
    }
    // validate (building.cpp:12-52): face and link references must resolve
    for (int w = 0; w < d->n_walls; ++w) {
        for (int k = 0; k < 2; ++k) {
            const hyg_face_attach& a = d->attach[2 * w + k];
            const int lim = a.kind == HYG_FACE_ZONE ? d->n_zones : d->n_channels;
            if (a.index < 0 || a.index >= lim || (a.kind != HYG_FACE_ZONE && a.kind != HYG_FACE_EXTERIOR)) {
                char m[160];
                std::snprintf(m, sizeof m, "wall %d face %d references %s %d which does not exist", w, k,
                              a.kind == HYG_FACE_ZONE ? "zone" : "channel", a.index);
                set_status(status, HYG_ESCHEMA, m);
                return HYG_ESCHEMA;
            }
        }
    }
    for (int z = 0; z < d->n_zones; ++z) {
        const hyg_zone_desc& zd = d->zones[z];
        for (int i = 0; i < zd.n_walls; ++i)
            if (zd.walls[i].wall < 0 || zd.walls[i].wall >= d->n_walls) {
                set_status(status, HYG_ESCHEMA, "zone links a wall which does not exist");
                return HYG_ESCHEMA;
            }
        for (int i = 0; i < zd.n_interzone; ++i)
            if (zd.interzone[i].peer < 0 || zd.interzone[i].peer >= d->n_zones) {
                set_status(status, HYG_ESCHEMA, "zone links a peer zone which does not exist");
                return HYG_ESCHEMA;
            }
        if (zd.sources < 0 || zd.sources >= d->n_zone_sources) {
            set_status(status, HYG_ESCHEMA, "zone references missing source schedules");
            return HYG_ESCHEMA;
        }
        for (int i = 0; i < zd.n_radiation; ++i) {
            const hyg_radiation_link& r = zd.radiation[i];
            if (r.emitter_wall < 0 || r.emitter_wall >= d->n_walls || r.receiver_wall < 0 ||
                r.receiver_wall >= d->n_walls) {
                set_status(status, HYG_ESCHEMA, "radiation link references a wall which does not exist");
                return HYG_ESCHEMA;
            }
        }
        if (zd.n_radiation > 0 && (!d->wall_thickness || !d->wall_k_TT0 || !(d->T_i > 0.0))) {
            set_status(status, HYG_EINVAL, "radiation needs wall_thickness, wall_k_TT0 and T_i");
            return HYG_EINVAL;
        }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        set_status(status, HYG_ECUDA, "no CUDA device (this library has no CPU fallback)");
        return HYG_ECUDA;
    }
    hyg_ctx* c = new hyg_ctx();
    c->device = d->device;
    if (cudaSetDevice(c->device) != cudaSuccess) {
        delete c;
        set_status(status, HYG_ECUDA, "cudaSetDevice failed");
        return HYG_ECUDA;
    }
    c->n_walls = d->n_walls;
    c->n = d->n_nodes;
    c->dx = d->dx;
    c->precision = d->precision;
    c->coeff_kind = d->coeff_kind;
    for (int i = 0; i < 4; ++i) c->p[i] = d->coeff_params[i];
    c->dt = d->dt;
    c->norm = d->divergence_norm > 0 ? d->divergence_norm : 1e3;
    c->eta_factor = d->eta_factor > 0 ? d->eta_factor : 1e-2;
    c->max_subiters = d->max_subiters > 0 ? d->max_subiters : 100;
    c->groups.resize(c->n_walls);
    c->biot.resize(2 * c->n_walls);
    c->attach.resize(2 * c->n_walls);
    std::vector<int> chan(2 * c->n_walls, 0);
    bool all_exterior = true;
    for (int w = 0; w < c->n_walls; ++w) {
        const hyg_wall_groups& g = d->groups[w];
        c->groups[w] = Groups{g.Fo_M, g.Fo_TT, g.Fo_TM, g.gamma};
        c->fo_m_pos = c->fo_m_pos && g.Fo_M > 0.0;
        for (int k = 0; k < 2; ++k) {
            const hyg_face_biot& b = d->biot[2 * w + k];
            c->biot[2 * w + k] = Biot{b.Bi_M, b.Bi_TT, b.Bi_TM};
            const hyg_face_attach& a = d->attach[2 * w + k];
            c->attach[2 * w + k] = Attach{a.kind, a.index};
            if (a.kind == HYG_FACE_EXTERIOR) chan[2 * w + k] = a.index;
            else all_exterior = false;
        }
    }
    c->channels.resize(d->n_channels);
    for (int i = 0; i < d->n_channels; ++i) {
        c->channels[i].u.set(d->channels[i].u_inf);
        c->channels[i].v.set(d->channels[i].v_inf);
        c->channels[i].g.set(d->channels[i].g_inf);
        c->channels[i].q.set(d->channels[i].q_inf);
    }
    for (int z = 0; z < d->n_zones; ++z) {
        const hyg_zone_desc& zd = d->zones[z];
        ZoneDev zz{};
        zz.kappa_a_tt1 = zd.kappa_a_tt1;
        zz.g_v = zd.g_v;
        zz.q_v1 = zd.q_v1;
        zz.q_v2 = zd.q_v2;
        zz.sign = zd.moisture_sign == HYG_MOISTURE_AS_PRINTED ? 1.0 : -1.0;
        zz.sources = zd.sources;
        zz.wall_begin = static_cast<int>(c->zlinks.size());
        for (int i = 0; i < zd.n_walls; ++i) {
            const hyg_zone_wall_link& l = zd.walls[i];
            c->zlinks.push_back(ZoneLinkDev{l.wall, l.face, l.Bi_M, l.Bi_TT, l.Bi_TM, l.theta_T, l.theta_M});
        }
        zz.wall_end = static_cast<int>(c->zlinks.size());
        zz.inz_begin = static_cast<int>(c->inz.size());
        for (int i = 0; i < zd.n_interzone; ++i) {
            const hyg_interzone_link& l = zd.interzone[i];
            c->inz.push_back(InzLinkDev{l.peer, l.g_inz, l.q_inz1, l.q_inz2});
        }
        zz.inz_end = static_cast<int>(c->inz.size());
        c->zones.push_back(zz);
    }
    c->zsrc.resize(3 * d->n_zone_sources);
    for (int i = 0; i < d->n_zone_sources; ++i) {
        c->zsrc[3 * i + 0].set(d->zone_sources[i].g_o);
        c->zsrc[3 * i + 1].set(d->zone_sources[i].q_o);
        c->zsrc[3 * i + 2].set(d->zone_sources[i].q_h);
    }
    c->out_u.set(d->outdoor_u);
    c->out_v.set(d->outdoor_v);
    c->src_tab.assign(d->n_zone_sources, TableHost{0, 3, {}});
    c->out_tab.width = 2;
    // per-wall coefficient models (BuildingWall::coeffs building.hpp:28)
    c->T_i = d->T_i;
    c->P_vi = d->P_vi;
    c->wall_kind.assign(c->n_walls, kCoeffConstant);
    std::vector<mat::Set> refs(c->n_walls, mat::Set{1, 1, 1, 1, 1, 1});
    for (int w = 0; w < c->n_walls; ++w) {
        if (d->coeff_kind == HYG_COEFF_ANALYTIC_D) c->wall_kind[w] = kCoeffAnalyticD;
        if (d->coeff_kind == HYG_COEFF_MATERIAL &&
            (!d->wall_coeff || d->wall_coeff[w] == HYG_COEFF_MATERIAL)) {
            c->wall_kind[w] = kCoeffMaterial;
            const hyg_coeff_set& r = d->wall_reference[w];
            refs[w] = mat::Set{r.c_M, r.k_M, r.c_TT, r.k_TT, r.c_TM, r.k_TM};
            c->any_material = true;
        }
        c->any_nonlinear = c->any_nonlinear || c->wall_kind[w] != kCoeffConstant;
    }
    // radiation CSR (radiation_fluxes building.cpp:88-105, zone_surface_u :77-86):
    // groups in zone / link order, bucketed by target face in that order
    struct RadGroup { int target; double num, den; std::vector<int64_t> e, r; std::vector<double> coef; };
    std::vector<RadGroup> rg;
    for (int z = 0; z < d->n_zones; ++z) {
        const hyg_zone_desc& zd = d->zones[z];
        if (zd.n_radiation == 0) continue;
        std::vector<int64_t> surf(c->n_walls, -1);      // last link of each wall in this zone wins
        for (int i = 0; i < zd.n_walls; ++i)
            surf[zd.walls[i].wall] = static_cast<int64_t>(zd.walls[i].wall) * c->n + (zd.walls[i].face == 0 ? 0 : c->n - 1);
        for (int i = 0; i < zd.n_walls; ++i) {
            const hyg_zone_wall_link& l = zd.walls[i];
            RadGroup g{2 * l.wall + (l.face == 0 ? 0 : 1), d->wall_thickness[l.wall], d->T_i * d->wall_k_TT0[l.wall], {}, {}, {}};
            for (int k = 0; k < zd.n_radiation; ++k) {
                const hyg_radiation_link& r = zd.radiation[k];
                if (r.receiver_wall != l.wall) continue;
                g.e.push_back(surf[r.emitter_wall]);
                g.r.push_back(surf[r.receiver_wall]);
                g.coef.push_back(r.view_factor * r.emissivity * 5.67e-8);   // PhysicalConstants::sigma
            }
            rg.push_back(std::move(g));
        }
    }
    std::stable_sort(rg.begin(), rg.end(), [](const RadGroup& x, const RadGroup& y) { return x.target < y.target; });
    std::vector<int> rad_tgt(2 * c->n_walls + 1, 0), rad_grp(1, 0);
    std::vector<double> rad_num, rad_den, rad_coef;
    std::vector<int64_t> rad_e, rad_r;
    for (const auto& g : rg) {
        rad_tgt[g.target + 1] += 1;
        rad_num.push_back(g.num);
        rad_den.push_back(g.den);
        for (size_t i = 0; i < g.e.size(); ++i) {
            rad_e.push_back(g.e[i]);
            rad_r.push_back(g.r[i]);
            rad_coef.push_back(g.coef[i]);
        }
        rad_grp.push_back(static_cast<int>(rad_e.size()));
    }
    for (int i = 0; i < 2 * c->n_walls; ++i) rad_tgt[i + 1] += rad_tgt[i];
    c->has_rad = !rg.empty();
    // K4 (k_ring.cuh): constant walls, face 0 exterior, face 1 on the wall's own
    // zone, W walls per zone in zone order, zone links = those walls' face 1,
    // inter-zone peers within +-1 on the ring, n in {64, 128, 256}, no radiation
    if (d->coeff_kind == HYG_COEFF_CONSTANT && d->precision == HYG_F64 && d->n_zones > 0 && !c->has_rad &&
        c->n_walls % d->n_zones == 0 && (c->n == 64 || c->n == 128 || c->n == 256)) {
        const int W = c->n_walls / d->n_zones, Z = d->n_zones;
        bool ok = W >= 1;
        for (int w = 0; ok && w < c->n_walls; ++w)
            ok = d->attach[2 * w].kind == HYG_FACE_EXTERIOR && d->attach[2 * w + 1].kind == HYG_FACE_ZONE &&
                 d->attach[2 * w + 1].index == w / W;
        for (int z = 0; ok && z < Z; ++z) {
            const hyg_zone_desc& zd = d->zones[z];
            ok = ok && zd.n_walls <= kRingMaxLinks && zd.n_interzone <= kRingMaxPeers;
            for (int i = 0; ok && i < zd.n_walls; ++i)
                ok = zd.walls[i].face == 1 && zd.walls[i].wall / W == z;
            for (int i = 0; ok && i < zd.n_interzone; ++i) {
                const int p = zd.interzone[i].peer;
                ok = p == (z + 1) % Z || p == (z - 1 + Z) % Z;
            }
        }
        if (ok) {
            const int npt = c->n / 16;
            int B = std::min(Z, 32 - 2 * kRingS);
            const int nch = std::max(1, d->n_channels), nsrc = d->n_zone_sources;
            auto fits = [&](int b) {
                const size_t sm = npt == 4 ? RingShape<4, kRingS>::smem_bytes(b, W, nch, nsrc)
                                  : npt == 8 ? RingShape<8, kRingS>::smem_bytes(b, W, nch, nsrc)
                                             : RingShape<16, kRingS>::smem_bytes(b, W, nch, nsrc);
                const int th = RingShape<8, kRingS>::threads(b, W);
                return sm <= 227u * 1024u && th <= 896;
            };
            while (B > 0 && !fits(B)) --B;
            if (B >= 1 && (npt == 4 || npt == 8)) {
                // K4r: the largest block whose roles fit 512 threads (128 registers each)
                int Br = std::min(Z, 32 - 2 * kRingRegS);
                auto fits_r = [&](int b) {
                    const int rw = RingShape<8, kRingS>::row_width(nch, nsrc);
                    return RingRegShape<8, kRingRegS>::threads(b, W) <= kRingRegThreads &&
                           RingRegShape<8, kRingRegS>::smem_doubles(b, W, c->n, rw) * sizeof(double) <= 227u * 1024u;
                };
                while (Br > 0 && !fits_r(Br)) --Br;
                c->ring_reg_B = Br;
                // K5: 128-node walls; the CTA's roles must fit its compiled size
                using SP = RingPipeShape<kRingPipeS>;
                int Bp = npt == 8 ? std::min(Z, SP::kB) : 0;
                auto fits_p = [&](int b) {
                    const int rw = RingShape<8, kRingS>::row_width(nch, nsrc);
                    return SP::threads(b, W) <= SP::kThreads && SP::local_zones(b) <= 32 &&
                           SP::smem_doubles(b, W, rw) * sizeof(double) <= 227u * 1024u;
                };
                while (Bp > 0 && !fits_p(Bp)) --Bp;
                c->ring_pipe_B = Bp;
                // K6 phase 1: LB local zones per CTA (LB - 2 S owned); about one CTA per
                // SM for long rings, never fewer than min(Z, 8) owned zones
                using SC = RingConeShape<kRingSplitS>;
                // the walls need their deepest stub's tail (26 nodes) inside the wall, the
                // forcing rows of a launch must fit both kernels' shared memory
                const size_t walls_smem = RingWallShape<8>::smem_doubles(kRingSplitS * kRingSplitMaxM, nch, kRingWallWarps) * sizeof(double);
                if (c->n >= RingConeShape<kRingSplitS>::kPS + kRingSplitS * (kRingSplitMaxM - 1) && walls_smem <= 100u * 1024u) {
                    const int rw = RingShape<8, kRingSplitS>::row_width(nch, nsrc);
                    int lb = 2 * kRingSplitS + 1;
                    while (SC::threads(lb + 1, W) <= kRingConeThreads &&
                           SC::smem_doubles(lb + 1, W, rw) * sizeof(double) <= 227u * 1024u)
                        ++lb;
                    if (SC::threads(lb, W) <= kRingConeThreads &&
                        SC::smem_doubles(lb, W, rw) * sizeof(double) <= 227u * 1024u) {
                        const int nsm = sm_count(c->device);
                        int ob = (Z + nsm - 1) / nsm;
                        ob = std::max(ob, std::min(Z, 8));
                        ob = std::min(ob, lb - 2 * kRingSplitS);
                        c->ring_cone_LB = ob + 2 * kRingSplitS;
                    }
                }
            }
            if (B >= 1) {
                c->ring = true;
                c->ring_W = W;
                c->ring_B = B;
            }
        }
    }
    c->fused = all_exterior && d->n_zones == 0 && d->coeff_kind == HYG_COEFF_CONSTANT && fused_grid(c->n);
    // the warp-register d(v) kernels take exp of x = -p2 (v - p3)^2 with fexp_addend,
    // valid for -700 <= x <= 0: every state inside their fast guard (|v| < 2) must
    // keep x in that range.  A growing exponential (p2 < 0) or a steeper one marches
    // on the per-step path with the full exp
    const double dv_reach = 2.0 + std::fabs(d->coeff_params[3]);
    const bool dv_neg = d->coeff_params[2] >= 0.0 && d->coeff_params[2] * dv_reach * dv_reach <= 700.0;
    c->nl_fused = all_exterior && d->n_zones == 0 && d->coeff_kind == HYG_COEFF_ANALYTIC_D && c->n <= 1024 &&
                  c->precision == HYG_F64 && dv_neg;
    c->tiled = all_exterior && d->n_zones == 0 && d->coeff_kind == HYG_COEFF_ANALYTIC_D && c->n > 1024 &&
               c->n_walls == 1 && c->precision == HYG_F64 && dv_neg;
    if (c->precision == HYG_F32 && !c->fused) {
        delete c;
        set_status(status, HYG_ENOTSUP, "fp32 state is implemented for exterior constant walls on fused grids only");
        return HYG_ENOTSUP;
    }
    if (c->precision == HYG_F32 && !(c->norm >= 3.0)) {
        delete c;
        set_status(status, HYG_ENOTSUP, "fp32 state needs divergence_norm >= 3");
        return HYG_ENOTSUP;
    }
    c->flux = false;
    for (const auto& ch : c->channels)
        if (!ch.flux_free()) c->flux = true;

    auto fail = [&](const char* m) {
        set_status(status, HYG_ECUDA, m);
        hyg_destroy(c);
        return HYG_ECUDA;
    };
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return fail("stream");
    c->own_stream = c->stream;
    if (const char* e = std::getenv("HYG_DEBUG_RING_SKIP")) c->ring_dbg_skip = std::atoi(e);   // timing only
    const size_t cells = static_cast<size_t>(c->cells());
    for (int b = 0; b < 2; ++b)
        for (int i = 0; i < 4; ++i) {
            if (cudaMalloc(&c->s64[b][i], cells * sizeof(double)) != cudaSuccess) return fail("state alloc");
            if (c->precision == HYG_F32 && cudaMalloc(&c->s32[b][i], cells * sizeof(float)) != cudaSuccess)
                return fail("state alloc");
        }
    // tensor maps of the state arrays (rows of 8 nodes, boxes of 32 rows): K3w's windows and,
    // for 128-node zone rings, K6's wall pairs
    if ((c->tiled && kTileNPT == 8) || (c->ring_cone_LB > 0 && c->n == 128)) {
        c->tmaps_ok = true;
        for (int b = 0; b < 2; ++b)
            for (int i = 0; i < 4; ++i)
                c->tmaps_ok = c->tmaps_ok && make_row_map(&c->tmaps[b].m[i], c->s64[b][i], static_cast<int64_t>(cells));
    }
    if (cudaMalloc(&c->d_groups, sizeof(Groups) * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_biot, sizeof(Biot) * 2 * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_attach, sizeof(Attach) * 2 * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_chan, sizeof(int) * 2 * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_coef, sizeof(WallCoef) * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&c->d_key, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_dom, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_wall_kind, sizeof(int) * c->n_walls) != cudaSuccess ||
        cudaMalloc(&c->d_ref, sizeof(mat::Set) * c->n_walls) != cudaSuccess)
        return fail("parameter alloc");
    cudaMemcpy(c->d_wall_kind, c->wall_kind.data(), sizeof(int) * c->n_walls, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_ref, refs.data(), sizeof(mat::Set) * c->n_walls, cudaMemcpyHostToDevice);
    cudaMemset(c->d_dom, 0xff, sizeof(unsigned long long));
    if (c->has_rad) {
        auto up = [&](auto*& dst, const auto& v) {
            using T = typename std::decay_t<decltype(v)>::value_type;
            if (cudaMalloc(&dst, sizeof(T) * std::max<size_t>(1, v.size())) != cudaSuccess) return false;
            if (!v.empty()) cudaMemcpy(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
            return true;
        };
        if (!up(c->d_rad_tgt, rad_tgt) || !up(c->d_rad_grp, rad_grp) || !up(c->d_rad_num, rad_num) ||
            !up(c->d_rad_den, rad_den) || !up(c->d_rad_coef, rad_coef) || !up(c->d_rad_e, rad_e) ||
            !up(c->d_rad_r, rad_r) || cudaMalloc(&c->d_qrad, sizeof(double) * 2 * c->n_walls) != cudaSuccess)
            return fail("radiation alloc");
    }
    cudaMemcpy(c->d_groups, c->groups.data(), sizeof(Groups) * c->n_walls, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_biot, c->biot.data(), sizeof(Biot) * 2 * c->n_walls, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_attach, c->attach.data(), sizeof(Attach) * 2 * c->n_walls, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_chan, chan.data(), sizeof(int) * 2 * c->n_walls, cudaMemcpyHostToDevice);
    const int nz = std::max<int>(1, static_cast<int>(c->zones.size()));
    for (int b = 0; b < 2; ++b)
        if (cudaMalloc(&c->zu[b], sizeof(double) * nz) != cudaSuccess ||
            cudaMalloc(&c->zv[b], sizeof(double) * nz) != cudaSuccess)
            return fail("zone alloc");
    if (!c->zones.empty()) {
        if (cudaMalloc(&c->d_zones, sizeof(ZoneDev) * c->zones.size()) != cudaSuccess ||
            cudaMalloc(&c->d_zlinks, sizeof(ZoneLinkDev) * std::max<size_t>(1, c->zlinks.size())) != cudaSuccess ||
            cudaMalloc(&c->d_inz, sizeof(InzLinkDev) * std::max<size_t>(1, c->inz.size())) != cudaSuccess)
            return fail("zone alloc");
        cudaMemcpy(c->d_zones, c->zones.data(), sizeof(ZoneDev) * c->zones.size(), cudaMemcpyHostToDevice);
        if (!c->zlinks.empty())
            cudaMemcpy(c->d_zlinks, c->zlinks.data(), sizeof(ZoneLinkDev) * c->zlinks.size(), cudaMemcpyHostToDevice);
        if (!c->inz.empty())
            cudaMemcpy(c->d_inz, c->inz.data(), sizeof(InzLinkDev) * c->inz.size(), cudaMemcpyHostToDevice);
        if (c->ring_reg_B > 0) {
            // K4r's per-zone parameter blocks (k_ring_reg.cuh), prefetched with the walls
            std::vector<double> zp(c->zones.size() * kRingZP, 0.0);
            c->ring_reg_small = true;
            for (const ZoneDev& d : c->zones)
                c->ring_reg_small = c->ring_reg_small && d.wall_end - d.wall_begin <= 6 && d.inz_end - d.inz_begin <= 2;
            if (!c->ring_reg_small) c->ring_pipe_B = 0;   // K5 walks exactly 6 link and 2 peer slots
            for (size_t z = 0; z < c->zones.size(); ++z) {
                const ZoneDev& d = c->zones[z];
                double* b = &zp[z * kRingZP];
                b[0] = 1.0 + d.kappa_a_tt1;
                b[1] = d.g_v;
                b[2] = d.q_v1;
                b[3] = d.q_v2;
                b[4] = d.wall_end - d.wall_begin;
                b[5] = d.inz_end - d.inz_begin;
                b[6] = d.sources;
                for (int q = 0; q < d.wall_end - d.wall_begin; ++q) {
                    const ZoneLinkDev& l = c->zlinks[d.wall_begin + q];
                    b[8 + 4 * q] = l.wall - static_cast<int>(z) * c->ring_W;
                    b[9 + 4 * q] = l.Bi_TT * l.theta_T;
                    b[10 + 4 * q] = l.Bi_TM * l.theta_T;
                    b[11 + 4 * q] = d.sign * l.Bi_M * l.theta_M;
                }
                for (int q = 0; q < d.inz_end - d.inz_begin; ++q) {
                    const InzLinkDev& l = c->inz[d.inz_begin + q];
                    b[40 + 4 * q] = l.peer;
                    b[41 + 4 * q] = l.g_inz;
                    b[42 + 4 * q] = l.q_inz1;
                    b[43 + 4 * q] = l.q_inz2;
                }
            }
            if (cudaMalloc(&c->d_ring_zp, sizeof(double) * zp.size()) != cudaSuccess) return fail("zone alloc");
            if (c->ring_cone_LB > 0) {
                const size_t Zn = c->zones.size();
                std::vector<double> zpT(zp.size());
                for (size_t z = 0; z < Zn; ++z)
                    for (int k = 0; k < kRingZP; ++k) zpT[k * Zn + z] = zp[z * kRingZP + k];
                constexpr int kTailMax = (RingConeShape<kRingSplitS>::kP + kRingSplitS * (kRingSplitMaxM - 2) + 1) & ~1;
                for (int b = 0; b < 2; ++b) {
                    for (int i = 0; i < 4; ++i)
                        if (cudaMalloc(&c->d_ring_tail[b][i], sizeof(double) * c->n_walls * kTailMax) != cudaSuccess)
                            return fail("zone alloc");
                    for (int i = 0; i < 2; ++i)
                        if (cudaMalloc(&c->d_ring_zt[b][i], sizeof(double) * Zn) != cudaSuccess) return fail("zone alloc");
                }
                if (cudaMalloc(&c->d_ring_series, sizeof(double) * Zn * kRingSplitS * kRingSplitMaxM * 2) != cudaSuccess ||
                    cudaMalloc(&c->d_ring_rowsT, sizeof(double) * 12 * c->n_walls) != cudaSuccess ||
                    cudaMalloc(&c->d_ring_zpT, sizeof(double) * zpT.size()) != cudaSuccess)
                    return fail("zone alloc");
                cudaMemcpy(c->d_ring_zpT, zpT.data(), sizeof(double) * zpT.size(), cudaMemcpyHostToDevice);
            }
            cudaMemcpy(c->d_ring_zp, zp.data(), sizeof(double) * zp.size(), cudaMemcpyHostToDevice);
        }
    }
    // WallField::uniform (wall.cpp:24-31) and ZoneState{} (zone.hpp:11-14): all 1
    {
        std::vector<double> ones(std::max<size_t>(cells, static_cast<size_t>(nz)), 1.0);
        for (int i = 0; i < 4; ++i)
            cudaMemcpy(c->s64[0][i], ones.data(), cells * sizeof(double), cudaMemcpyHostToDevice);
        cudaMemcpy(c->zu[0], ones.data(), sizeof(double) * nz, cudaMemcpyHostToDevice);
        cudaMemcpy(c->zv[0], ones.data(), sizeof(double) * nz, cudaMemcpyHostToDevice);
    }
    for (auto& e : c->ev) cudaEventCreate(&e);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail("init");
    hyg_status tmp;
    if (to_f32(c, &tmp) != HYG_OK) return fail("init f32");
    *out = c;
    return HYG_OK;
}

void hyg_destroy(hyg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    drain_pending(c);
    for (int b = 0; b < 2; ++b) {
        for (int i = 0; i < 4; ++i) {
            cudaFree(c->s64[b][i]);
            cudaFree(c->s32[b][i]);
        }
        cudaFree(c->zu[b]);
        cudaFree(c->zv[b]);
    }
    for (int i = 0; i < 4; ++i) cudaFree(c->snap[i]);
    cudaFree(c->snap_z[0]);
    cudaFree(c->snap_z[1]);
    cudaFree(c->d_groups);
    cudaFree(c->d_biot);
    cudaFree(c->d_attach);
    cudaFree(c->d_chan);
    cudaFree(c->d_coef);
    cudaFree(c->d_zones);
    cudaFree(c->d_zlinks);
    cudaFree(c->d_inz);
    cudaFree(c->d_ring_zp);
    cudaFree(c->d_ring_series);
    for (int b = 0; b < 2; ++b) {
        for (int i = 0; i < 4; ++i) cudaFree(c->d_ring_tail[b][i]);
        for (int i = 0; i < 2; ++i) cudaFree(c->d_ring_zt[b][i]);
    }
    cudaFree(c->d_ring_rowsT);
    cudaFree(c->d_ring_zpT);
    cudaFree(c->d_table);
    cudaFree(c->d_boot);
    cudaFree(c->d_src);
    cudaFree(c->d_flag);
    cudaFree(c->d_key);
    cudaFree(c->d_dom);
    cudaFree(c->d_wall_kind);
    cudaFree(c->d_ref);
    cudaFree(c->d_star);
    cudaFree(c->d_impl);
    for (void* q : {static_cast<void*>(c->d_rad_tgt), static_cast<void*>(c->d_rad_grp),
                    static_cast<void*>(c->d_rad_num), static_cast<void*>(c->d_rad_den),
                    static_cast<void*>(c->d_rad_coef), static_cast<void*>(c->d_qrad),
                    static_cast<void*>(c->d_rad_e), static_cast<void*>(c->d_rad_r)})
        cudaFree(q);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

int hyg_set_state(hyg_ctx* c, const double* up, const double* uc, const double* vp, const double* vc,
                  const double* zu, const double* zv, double t_star, int64_t layer) {
    hyg_status* status = nullptr;
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    const size_t bytes = static_cast<size_t>(c->cells()) * sizeof(double);
    const double* src[4] = {up, uc, vp, vc};
    for (int i = 0; i < 4; ++i)
        if (src[i]) HYG_CUDA(cudaMemcpyAsync(c->s64[c->cur][i], src[i], bytes, cudaMemcpyHostToDevice, c->stream));
    if (!c->zones.empty()) {
        const size_t zb = c->zones.size() * sizeof(double);
        if (zu) HYG_CUDA(cudaMemcpyAsync(c->zu[c->zcur], zu, zb, cudaMemcpyHostToDevice, c->stream));
        if (zv) HYG_CUDA(cudaMemcpyAsync(c->zv[c->zcur], zv, zb, cudaMemcpyHostToDevice, c->stream));
    }
    c->t = t_star;
    c->layer = layer;
    hyg_status tmp;
    int rc = to_f32(c, &tmp);
    if (rc) return rc;
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int hyg_get_state(hyg_ctx* c, double* up, double* uc, double* vp, double* vc, double* zu, double* zv,
                  double* t_star, int64_t* layer) {
    hyg_status* status = nullptr;
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    hyg_status tmp;
    int rc = from_f32(c, &tmp);
    if (rc) return rc;
    const size_t bytes = static_cast<size_t>(c->cells()) * sizeof(double);
    double* dst[4] = {up, uc, vp, vc};
    for (int i = 0; i < 4; ++i)
        if (dst[i]) HYG_CUDA(cudaMemcpyAsync(dst[i], c->s64[c->cur][i], bytes, cudaMemcpyDeviceToHost, c->stream));
    if (!c->zones.empty()) {
        const size_t zb = c->zones.size() * sizeof(double);
        if (zu) HYG_CUDA(cudaMemcpyAsync(zu, c->zu[c->zcur], zb, cudaMemcpyDeviceToHost, c->stream));
        if (zv) HYG_CUDA(cudaMemcpyAsync(zv, c->zv[c->zcur], zb, cudaMemcpyDeviceToHost, c->stream));
    }
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    if (t_star) *t_star = c->t;
    if (layer) *layer = c->layer;
    return HYG_OK;
}

int hyg_get_cells(hyg_ctx* c, int64_t cell0, int64_t count, double* up, double* uc, double* vp,
                  double* vc) {
    hyg_status* status = nullptr;
    if (!c || cell0 < 0 || count < 0 || cell0 + count > c->cells()) return HYG_EINVAL;
    if (c->precision != HYG_F64) return HYG_ENOTSUP;
    cudaSetDevice(c->device);
    double* dst[4] = {up, uc, vp, vc};
    for (int i = 0; i < 4; ++i)
        if (dst[i])
            HYG_CUDA(cudaMemcpyAsync(dst[i], c->s64[c->cur][i] + cell0, count * sizeof(double),
                                     cudaMemcpyDefault, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int hyg_set_cells(hyg_ctx* c, int64_t cell0, int64_t count, const double* up, const double* uc,
                  const double* vp, const double* vc) {
    hyg_status* status = nullptr;
    if (!c || cell0 < 0 || count < 0 || cell0 + count > c->cells()) return HYG_EINVAL;
    if (c->precision != HYG_F64) return HYG_ENOTSUP;
    cudaSetDevice(c->device);
    const double* src[4] = {up, uc, vp, vc};
    for (int i = 0; i < 4; ++i)
        if (src[i])
            HYG_CUDA(cudaMemcpyAsync(c->s64[c->cur][i] + cell0, src[i], count * sizeof(double),
                                     cudaMemcpyDefault, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int hyg_get_zones(hyg_ctx* c, int32_t z0, int32_t count, double* zu, double* zv) {
    hyg_status* status = nullptr;
    if (!c || z0 < 0 || count < 0 || z0 + count > static_cast<int>(c->zones.size())) return HYG_EINVAL;
    cudaSetDevice(c->device);
    if (zu) HYG_CUDA(cudaMemcpyAsync(zu, c->zu[c->zcur] + z0, count * sizeof(double), cudaMemcpyDefault, c->stream));
    if (zv) HYG_CUDA(cudaMemcpyAsync(zv, c->zv[c->zcur] + z0, count * sizeof(double), cudaMemcpyDefault, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int hyg_set_zones(hyg_ctx* c, int32_t z0, int32_t count, const double* zu, const double* zv) {
    hyg_status* status = nullptr;
    if (!c || z0 < 0 || count < 0 || z0 + count > static_cast<int>(c->zones.size())) return HYG_EINVAL;
    cudaSetDevice(c->device);
    if (zu) HYG_CUDA(cudaMemcpyAsync(c->zu[c->zcur] + z0, zu, count * sizeof(double), cudaMemcpyDefault, c->stream));
    if (zv) HYG_CUDA(cudaMemcpyAsync(c->zv[c->zcur] + z0, zv, count * sizeof(double), cudaMemcpyDefault, c->stream));
    HYG_CUDA(cudaStreamSynchronize(c->stream));
    return HYG_OK;
}

int hyg_set_owned(hyg_ctx* c, int64_t cell0, int64_t cell1, int32_t zone0, int32_t zone1,
                  hyg_reduce_fn reduce, void* user) {
    if (!c || cell0 < 0 || cell1 < cell0 || zone0 < 0 || zone1 < zone0) return HYG_EINVAL;
    c->own_c0 = cell0;
    c->own_c1 = cell1;
    c->own_z0 = zone0;
    c->own_z1 = zone1;
    c->reduce = reduce;
    c->reduce_user = user;
    // K1/K2 guard every wall: a wall-batch shard with partial ownership marches
    // on the per-step path, whose guard honours the owned range.  K3 (one long
    // wall) stays: its fast guard only decides whether to replay on the
    // per-step path, which then applies the owned range exactly.
    if (cell0 > 0 || cell1 < c->cells()) c->fused = c->nl_fused = false;
    // the zone-ring kernels (K5/K4r/K4) guard whole blocks, halo copies
    // included: a shard keeps them (every owned value is exact), and a flagged
    // launch is replayed on the per-step path, whose guard honours the owned
    // ranges (advance_ring)
    c->owned_partial = cell0 > 0 || cell1 < c->cells() || zone0 > 0 || zone1 < static_cast<int>(c->zones.size());
    return HYG_OK;
}

int hyg_snapshot(hyg_ctx* c) {
    hyg_status* status = nullptr;
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    const size_t es = c->precision == HYG_F32 ? sizeof(float) : sizeof(double);
    const size_t bytes = static_cast<size_t>(c->cells()) * es;
    const size_t nz = std::max<size_t>(1, c->zones.size());
    for (int i = 0; i < 4; ++i) {
        if (!c->snap[i]) HYG_CUDA(cudaMalloc(&c->snap[i], bytes));
        const void* src = c->precision == HYG_F32 ? static_cast<const void*>(c->s32[c->cur][i])
                                                  : static_cast<const void*>(c->s64[c->cur][i]);
        HYG_CUDA(cudaMemcpyAsync(c->snap[i], src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    }
    for (int i = 0; i < 2; ++i) {
        if (!c->snap_z[i]) HYG_CUDA(cudaMalloc(&c->snap_z[i], nz * sizeof(double)));
        HYG_CUDA(cudaMemcpyAsync(c->snap_z[i], i ? c->zv[c->zcur] : c->zu[c->zcur], nz * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    c->snap_t = c->t;
    c->snap_layer = c->layer;
    return HYG_OK;
}

int hyg_restore(hyg_ctx* c) {
    hyg_status* status = nullptr;
    if (!c || c->snap_layer < 0) return HYG_EINVAL;
    cudaSetDevice(c->device);
    const size_t es = c->precision == HYG_F32 ? sizeof(float) : sizeof(double);
    const size_t bytes = static_cast<size_t>(c->cells()) * es;
    const size_t nz = std::max<size_t>(1, c->zones.size());
    for (int i = 0; i < 4; ++i) {
        void* dst = c->precision == HYG_F32 ? static_cast<void*>(c->s32[c->cur][i])
                                            : static_cast<void*>(c->s64[c->cur][i]);
        HYG_CUDA(cudaMemcpyAsync(dst, c->snap[i], bytes, cudaMemcpyDeviceToDevice, c->stream));
    }
    for (int i = 0; i < 2; ++i)
        HYG_CUDA(cudaMemcpyAsync(i ? c->zv[c->zcur] : c->zu[c->zcur], c->snap_z[i], nz * sizeof(double),
                                 cudaMemcpyDeviceToDevice, c->stream));
    c->t = c->snap_t;
    c->layer = c->snap_layer;
    return HYG_OK;
}

int hyg_set_channel_table(hyg_ctx* c, int32_t channel, int64_t first_layer, int64_t n_layers,
                          const hyg_ambient* values) {
    if (!c || channel < 0 || channel >= static_cast<int>(c->channels.size()) || n_layers < 0 ||
        (n_layers > 0 && !values))
        return HYG_EINVAL;
    ChannelHost& ch = c->channels[channel];
    ch.tab_first = first_layer;
    ch.tab.assign(values, values + n_layers);
    ++c->gen;
    c->flux = false;
    for (const auto& x : c->channels)
        if (!x.flux_free()) c->flux = true;
    return HYG_OK;
}

int hyg_set_source_table(hyg_ctx* c, int32_t source, int64_t first_layer, int64_t n_layers,
                         const double* values) {
    if (!c || source < 0 || source >= static_cast<int>(c->src_tab.size()) || n_layers < 0 ||
        (n_layers > 0 && !values))
        return HYG_EINVAL;
    c->src_tab[source] = TableHost{first_layer, 3, std::vector<double>(values, values + 3 * n_layers)};
    return HYG_OK;
}

int hyg_set_outdoor_table(hyg_ctx* c, int64_t first_layer, int64_t n_layers, const double* values) {
    if (!c || n_layers < 0 || (n_layers > 0 && !values)) return HYG_EINVAL;
    c->out_tab = TableHost{first_layer, 2, std::vector<double>(values, values + 2 * n_layers)};
    return HYG_OK;
}

int hyg_bootstrap(hyg_ctx* c, int32_t kind, hyg_status* status) {
    clear_status(status);
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    if (kind != HYG_BOOT_IMPLICIT && kind != HYG_BOOT_EXPLICIT) {
        set_status(status, HYG_EINVAL, "unknown bootstrap kind");
        return HYG_EINVAL;
    }
    int rc = from_f32(c, status);
    if (rc) return rc;
    // forcing: explicit step at layer-n time, implicit step at t^{n+1} (building.cpp:196)
    const double t_force = kind == HYG_BOOT_EXPLICIT ? c->t : c->t + c->dt;
    {   // one ambient row, kept apart from the cached per-layer table
        const int64_t lay = c->layer + (kind == HYG_BOOT_EXPLICIT ? 0 : 1);
        const int nch = std::max<int>(1, static_cast<int>(c->channels.size()));
        c->h_boot.assign(nch, Ambient{1, 1, 0, 0});
        for (int ch = 0; ch < static_cast<int>(c->channels.size()); ++ch)
            c->h_boot[ch] = c->channels[ch].at(lay, t_force);
        if (!c->d_boot) HYG_CUDA(cudaMalloc(&c->d_boot, sizeof(Ambient) * nch));
        HYG_CUDA(cudaMemcpyAsync(c->d_boot, c->h_boot.data(), sizeof(Ambient) * nch, cudaMemcpyHostToDevice,
                                 c->stream));
    }
    const int nsrc = static_cast<int>(c->zsrc.size() / 3);
    if (!c->zones.empty()) {
        std::vector<double> tf{t_force};
        rc = upload_src(c, c->layer + (kind == HYG_BOOT_EXPLICIT ? 0 : 1), tf, status);
        if (rc) return rc;
    }
    HYG_CUDA(cudaMemsetAsync(c->d_key, 0xff, sizeof(unsigned long long), c->stream));
    StepArgs a = step_args(c, c->cur, c->dt);
    a.amb = c->d_boot;
    int passes = 0;
    a.star.node = a.star.half = nullptr;     // no tables unless built below
    if (kind == HYG_BOOT_EXPLICIT) {
        // euler_explicit_step per wall (wall.cpp:266-317); with zones this is the
        // reference's EulerExplicit building step (building.cpp:174-183)
        if (c->has_rad) launch_radiation(c, a.in[1]);
        if (c->any_material) {      // clamped tables of layer n (wall.cpp:271)
            rc = launch_star_tables(c, a.in[1], a.in[3], false, c->layer, status);
            if (rc) return rc;
            a.star = StarTab{c->d_star, c->d_star + 6 * c->cells(), c->cells()};
        }
        {
            LaunchScope ls(c, "explicit_boot", static_cast<double>(c->cells()));
            k_explicit_boot<<<static_cast<int>((c->cells() + 255) / 256), 256, 0, c->stream>>>(a);
        }
        if (!c->zones.empty()) {
            ZoneArgs z{};
            z.n_zones = static_cast<int>(c->zones.size());
            z.n = c->n;
            z.dt = c->dt;
            z.zones = c->d_zones;
            z.links = c->d_zlinks;
            z.inz = c->d_inz;
            z.src = c->d_src;
            z.n_sources = nsrc;
            z.uc = c->s64[c->cur][1];
            z.vc = c->s64[c->cur][3];
            z.zu_in = c->zu[c->zcur];
            z.zv_in = c->zv[c->zcur];
            z.zu_out = c->zu[1 - c->zcur];
            z.zv_out = c->zv[1 - c->zcur];
            z.layer = c->layer;
            z.norm = c->norm;
            z.fail_key = c->d_key;
                z.own0 = c->own_z0;
                z.own1 = c->own_z1;
            LaunchScope ls(c, "zone_step", 0.0);
            k_zone_step<<<(z.n_zones + 127) / 128, 128, 0, c->stream>>>(z);
            c->zcur ^= 1;
        }
    } else {
        // step_implicit (building.cpp:189-268): walls and zones iterated jointly
        // until the max-norm change of every wall node and zone scalar < eta
        const double eta = c->eta_factor * c->dt;
        const size_t cells = static_cast<size_t>(c->cells());
        const int nz = std::max<int>(1, static_cast<int>(c->zones.size()));
        double* scr = nullptr;
        double* zit = nullptr;         // zone iterates: [4][nz] = (u,v) x (snapshot, new)
        unsigned long long* d_diff = nullptr;
        // scratch kept for the context's lifetime: a stream-ordered free hands the
        // pages back to the driver and the next start would map them again
        if (!c->d_impl) {
            HYG_CUDA(cudaMalloc(&c->d_impl, sizeof(double) * (5 * cells + 4 * static_cast<size_t>(nz)) +
                                                sizeof(unsigned long long)));
        }
        scr = c->d_impl;
        zit = c->d_impl + 5 * cells;
        d_diff = reinterpret_cast<unsigned long long*>(zit + 4 * nz);
        // iterates start from layer n (building.cpp:200-206)
        HYG_CUDA(cudaMemcpyAsync(a.out[1], a.in[1], cells * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        HYG_CUDA(cudaMemcpyAsync(a.out[3], a.in[3], cells * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        HYG_CUDA(cudaMemcpyAsync(zit, c->zu[c->zcur], nz * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        HYG_CUDA(cudaMemcpyAsync(zit + nz, c->zv[c->zcur], nz * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        int snap = 0;                  // zit[snap*2*nz ...] is the snapshot
        double diff = 0.0;
        int rcl = HYG_OK;
        for (;;) {
            ++passes;
            HYG_CUDA(cudaMemsetAsync(d_diff, 0, sizeof(unsigned long long), c->stream));
            HYG_CUDA(cudaMemsetAsync(c->d_key, 0xff, sizeof(unsigned long long), c->stream));
            double* zs_u = zit + snap * 2 * nz;
            double* zs_v = zs_u + nz;
            double* zn_u = zit + (1 - snap) * 2 * nz;
            double* zn_v = zn_u + nz;
            a.zu = zs_u;
            a.zv = zs_v;
            // radiation refreshed from the iterate surfaces (building.cpp:212), clamped
            // tables of the iterate for the nonlinear walls (wall.cpp:450)
            if (c->has_rad) launch_radiation(c, a.out[1]);
            if (c->any_nonlinear) {
                rc = launch_star_tables(c, a.out[1], a.out[3], false, c->layer, status);
                if (rc) return rc;
                a.star = StarTab{c->d_star, c->d_star + 6 * c->cells(), c->cells()};
                LaunchScope ls(c, "implicit_table_pass", static_cast<double>(c->cells()));
                k_implicit_table_pass<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(a, scr, d_diff);
            }
            {
                LaunchScope ls(c, "implicit_unit_pass", static_cast<double>(c->cells()));
                k_implicit_unit_pass<<<(c->n_walls + 127) / 128, 128, 0, c->stream>>>(a, scr, d_diff);
            }
            if (!c->zones.empty()) {
                ZoneImplicitArgs z{};
                z.n_zones = static_cast<int>(c->zones.size());
                z.n = c->n;
                z.dt = c->dt;
                z.zones = c->d_zones;
                z.links = c->d_zlinks;
                z.inz = c->d_inz;
                z.src = c->d_src;
                z.n_sources = nsrc;
                z.wu = a.out[1];
                z.wv = a.out[3];
                z.zu_n = c->zu[c->zcur];
                z.zv_n = c->zv[c->zcur];
                z.zu_s = zs_u;
                z.zv_s = zs_v;
                z.zu_out = zn_u;
                z.zv_out = zn_v;
                z.layer = c->layer;
                z.norm = c->norm;
                z.diff = d_diff;
                z.fail_key = c->d_key;
                z.own0 = c->own_z0;
                z.own1 = c->own_z1;
                LaunchScope ls(c, "zone_implicit", 0.0);
                k_zone_implicit<<<(z.n_zones + 127) / 128, 128, 0, c->stream>>>(z);
                snap ^= 1;
            }
            HYG_CUDA(cudaGetLastError());
            unsigned long long bits = 0;
            HYG_CUDA(cudaMemcpyAsync(&bits, d_diff, sizeof bits, cudaMemcpyDeviceToHost, c->stream));
            HYG_CUDA(cudaStreamSynchronize(c->stream));
            std::memcpy(&diff, &bits, sizeof diff);
            if (c->reduce) diff = c->reduce(c->reduce_user, diff);   // joint residual over shards
            if (diff < eta) break;
            if (passes >= c->max_subiters) {
                rcl = HYG_ECONVERGE;
                break;
            }
        }
        if (rcl == HYG_OK && !c->zones.empty()) {
            // zone states := the converged iterate (last written = current snapshot)
            HYG_CUDA(cudaMemcpyAsync(c->zu[1 - c->zcur], zit + snap * 2 * nz, nz * sizeof(double),
                                     cudaMemcpyDeviceToDevice, c->stream));
            HYG_CUDA(cudaMemcpyAsync(c->zv[1 - c->zcur], zit + snap * 2 * nz + nz, nz * sizeof(double),
                                     cudaMemcpyDeviceToDevice, c->stream));
            c->zcur ^= 1;
        }
        if (rcl != HYG_OK) {
            HYG_CUDA(cudaStreamSynchronize(c->stream));
            if (status) {
                status->code = HYG_ECONVERGE;
                status->residual = diff;
                status->subiterations = passes;
                std::snprintf(status->message, sizeof status->message,
                              "building fixed point did not converge in %d sub-iterations at t* = %.17g "
                              "(residual %.17g)", c->max_subiters, c->t + c->dt, diff);
            }
            to_f32(c, nullptr);
            return HYG_ECONVERGE;
        }
    }
    HYG_CUDA(cudaGetLastError());
    c->cur ^= 1;
    unsigned long long key;
    rc = read_key(c, &key, status);
    if (rc) return rc;
    c->t = c->t + c->dt;
    c->layer += 1;
    if (status) status->subiterations = passes;
    rc = to_f32(c, status);
    if (rc) return rc;
    if (key != ~0ull) return diverged(c, key, status);
    return HYG_OK;
}

int hyg_advance_overlapped(hyg_ctx* c, int64_t nsteps, double dt, int64_t edge_lo, int64_t edge_hi, void* event,
                           hyg_status* status) {
    if (!c || nsteps < 0 || edge_lo < 0 || edge_hi < 0) return HYG_EINVAL;
    if (!event) return hyg_advance(c, nsteps, dt, status);
    cudaSetDevice(c->device);
    const double dte = dt > 0.0 ? dt : c->dt;
    if (nsteps > 0 && c->tiled && dte > 0.0 && c->fo_m_pos && c->norm >= 2.0) {
        c->ov_lo = edge_lo;                   // consumed by advance_tiled's first launch
        c->ov_hi = edge_hi;
        c->ov_event = static_cast<cudaEvent_t>(event);
    } else if (cudaStreamWaitEvent(c->stream, static_cast<cudaEvent_t>(event), 0) != cudaSuccess) {
        return HYG_ECUDA;                     // every other path: behind the refresh, no overlap
    }
    const int rc = hyg_advance(c, nsteps, dt, status);
    c->ov_event = nullptr;
    return rc;
}

int hyg_advance(hyg_ctx* c, int64_t nsteps, double dt, hyg_status* status) {
    clear_status(status);
    if (!c || nsteps < 0) return HYG_EINVAL;
    if (nsteps == 0) return HYG_OK;
    cudaSetDevice(c->device);
    if (!(dt > 0.0)) dt = c->dt;
    int rc = c->fused      ? advance_fused(c, nsteps, dt, status)
             // the warp-register d(v) kernels scale the half-node coefficients by
             // 2 Fo_M dt/dx^2 (k_dv_warp.cuh): they need it positive
             : c->nl_fused && dt > 0.0 && c->fo_m_pos ? advance_nonlinear(c, nsteps, dt, status)
             : c->tiled && dt > 0.0 && c->fo_m_pos    ? advance_tiled(c, nsteps, dt, status)
             : c->ring     ? advance_ring(c, nsteps, dt, status)
                           : advance_general(c, nsteps, dt, status);
    if (status && rc == HYG_OK) status->code = HYG_OK;
    return rc;
}

int hyg_run(hyg_ctx* c, double horizon, double cadence, int32_t boot_kind, hyg_frame_fn frame,
            void* user, hyg_status* status) {
    clear_status(status);
    if (!c) return HYG_EINVAL;
    if (!(horizon >= 0.0)) {   // validate building.cpp:13
        set_status(status, HYG_ESCHEMA, "horizon must be non-negative");
        return HYG_ESCHEMA;
    }
    const int64_t nsteps = std::llround(horizon / c->dt);
    // lround of a huge cadence overflows in the reference (UB); here a cadence
    // beyond the horizon means initial and final frames only
    const double strides = cadence / c->dt;
    const int64_t stride = !(strides < 4.0e18) ? nsteps + 1 : std::max<int64_t>(1, std::llround(strides));
    if (frame) frame(user, c->layer, c->t, c);
    int64_t done = 0;
    int boot_passes = 0;
    if (nsteps > 0) {
        const int rc = hyg_bootstrap(c, boot_kind, status);
        if (rc) return rc;
        boot_passes = status ? status->subiterations : 0;
        ++done;
        if (frame && (done % stride == 0 || done == nsteps)) frame(user, c->layer, c->t, c);
    }
    while (done < nsteps) {
        const int64_t chunk = std::min(stride - done % stride, nsteps - done);
        const int rc = hyg_advance(c, chunk, c->dt, status);
        if (rc) return rc;
        done += chunk;
        if (frame && (done % stride == 0 || done == nsteps)) frame(user, c->layer, c->t, c);
    }
    if (status) status->subiterations = boot_passes;   // SimulationResult::bootstrap_subiters
    return HYG_OK;
}

int hyg_run_scheme(hyg_ctx* c, int32_t scheme, double horizon, double cadence, hyg_frame_fn frame, void* user,
                   hyg_run_report* report, hyg_status* status) {
    clear_status(status);
    if (!c) return HYG_EINVAL;
    if (report) *report = hyg_run_report{0, 0, 0, 0.0};
    if (scheme != HYG_SCHEME_DF && scheme != HYG_SCHEME_EULER_IMPLICIT && scheme != HYG_SCHEME_EULER_EXPLICIT) {
        set_status(status, HYG_EINVAL, "unknown scheme");
        return HYG_EINVAL;
    }
    if (!(horizon >= 0.0)) {   // validate building.cpp:13
        set_status(status, HYG_ESCHEMA, "horizon must be non-negative");
        return HYG_ESCHEMA;
    }
    const int64_t nsteps = std::llround(horizon / c->dt);
    const double strides = cadence / c->dt;
    const int64_t stride = !(strides < 4.0e18) ? nsteps + 1 : std::max<int64_t>(1, std::llround(strides));
    if (frame) frame(user, c->layer, c->t, c);
    int64_t done = 0;
    int64_t subiter_sum = 0;
    int max_seen = 0, boot = 0;
    const int64_t layer0 = c->layer;
    auto finish = [&](int rc) {
        // SimulationResult::steps counts the steps completed before a failure
        // (building.cpp:339-341): the failing step (output layer st.layer) is not
        if (rc != HYG_OK && status && status->layer > layer0) done = status->layer - 1 - layer0;
        if (report) {
            report->steps = done;
            report->bootstrap_subiters = boot;
            report->max_subiters_seen = max_seen;
            const int64_t counted = scheme == HYG_SCHEME_DF ? std::max<int64_t>(done - 1, 0) : done;
            report->mean_subiters = counted > 0 ? static_cast<double>(subiter_sum) / counted : 0.0;
        }
        return rc;
    };
    if (scheme == HYG_SCHEME_DF && nsteps > 0) {     // DF: implicit start counted as step 1
        const int rc = hyg_bootstrap(c, HYG_BOOT_IMPLICIT, status);
        if (rc) return finish(rc);
        boot = status ? status->subiterations : 0;
        ++done;
        if (frame && (done % stride == 0 || done == nsteps)) frame(user, c->layer, c->t, c);
    }
    while (done < nsteps) {
        if (scheme == HYG_SCHEME_DF) {
            const int64_t chunk = std::min(stride - done % stride, nsteps - done);
            const int rc = hyg_advance(c, chunk, c->dt, status);
            if (rc) return finish(rc);
            done += chunk;              // DF steps report 0 subiterations
        } else {
            // step_implicit / step_explicit(EulerExplicit) per step (building.cpp:327-331),
            // each guarded like the DF steps
            hyg_status st{};
            const int rc = hyg_bootstrap(c, scheme == HYG_SCHEME_EULER_IMPLICIT ? HYG_BOOT_IMPLICIT
                                                                                : HYG_BOOT_EXPLICIT, &st);
            if (status) *status = st;
            if (rc) return finish(rc);
            subiter_sum += st.subiterations;
            max_seen = std::max(max_seen, static_cast<int>(st.subiterations));
            ++done;
        }
        if (frame && (done % stride == 0 || done == nsteps)) frame(user, c->layer, c->t, c);
    }
    if (status) status->subiterations = boot;
    return finish(HYG_OK);
}

int hyg_synchronize(hyg_ctx* c) {
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return HYG_ECUDA;
    drain_pending(c);
    return HYG_OK;
}

int hyg_host_register(void* ptr, size_t bytes) {
    return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? HYG_OK : HYG_ECUDA;
}
int hyg_host_unregister(void* ptr) { return cudaHostUnregister(ptr) == cudaSuccess ? HYG_OK : HYG_ECUDA; }

int hyg_event_record(hyg_ctx* c, int32_t slot) {
    if (!c || slot < 0 || slot >= 16) return HYG_EINVAL;
    return cudaEventRecord(c->ev[slot], c->stream) == cudaSuccess ? HYG_OK : HYG_ECUDA;
}

int hyg_event_elapsed_ms(hyg_ctx* c, int32_t a, int32_t b, double* ms) {
    if (!c || a < 0 || a >= 16 || b < 0 || b >= 16 || !ms) return HYG_EINVAL;
    if (cudaEventSynchronize(c->ev[b]) != cudaSuccess) return HYG_ECUDA;
    float f = 0.f;
    if (cudaEventElapsedTime(&f, c->ev[a], c->ev[b]) != cudaSuccess) return HYG_ECUDA;
    *ms = f;
    return HYG_OK;
}

int hyg_set_profiling(hyg_ctx* c, int32_t on) {
    if (!c) return HYG_EINVAL;
    c->profiling = on != 0;
    return HYG_OK;
}
int hyg_kernel_stats_count(hyg_ctx* c) {
    if (!c) return 0;
    hyg_synchronize(c);
    return static_cast<int>(c->stats.size());
}
int hyg_kernel_stats(hyg_ctx* c, int32_t i, const char** name, int64_t* launches, double* ms,
                     double* updates) {
    if (!c || i < 0 || i >= static_cast<int>(c->stats.size())) return HYG_EINVAL;
    const Stat& s = c->stats[i];
    if (name) *name = s.name.c_str();
    if (launches) *launches = s.launches;
    if (ms) *ms = s.ms;
    if (updates) *updates = s.updates;
    return HYG_OK;
}
int hyg_set_stream(hyg_ctx* c, void* stream) {
    if (!c) return HYG_EINVAL;
    cudaSetDevice(c->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    if (s != c->stream) {
        // order the new stream after everything issued so far on the old one
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return HYG_ECUDA;
        cudaEventRecord(e, c->stream);
        cudaStreamWaitEvent(s, e, 0);
        cudaEventDestroy(e);
        c->stream = s;
    }
    return HYG_OK;
}

int hyg_set_exchange_stream(hyg_ctx* c, void* stream) {
    if (!c) return HYG_EINVAL;
    c->xstream = static_cast<cudaStream_t>(stream);
    return HYG_OK;
}

int hyg_pack_cells(hyg_ctx* c, int64_t cell0, int64_t count, double* buf) {
    if (!c || cell0 < 0 || count < 0 || cell0 + count > c->cells() || (count > 0 && !buf)) return HYG_EINVAL;
    if (c->precision != HYG_F64) return HYG_ENOTSUP;
    if (count == 0) return HYG_OK;
    cudaSetDevice(c->device);
    Layers4 L{{c->s64[c->cur][0], c->s64[c->cur][1], c->s64[c->cur][2], c->s64[c->cur][3]}};
    const int grid = static_cast<int>(std::min<int64_t>((4 * count + 255) / 256, 4 * sm_count(c->device)));
    {
        LaunchScope ls(c, "pack_cells", 0.0);
        k_pack_cells<<<grid, 256, 0, c->xstream ? c->xstream : c->stream>>>(L, cell0, count, buf);
    }
    return cudaGetLastError() == cudaSuccess ? HYG_OK : HYG_ECUDA;
}

int hyg_unpack_cells(hyg_ctx* c, int64_t cell0, int64_t count, const double* buf) {
    if (!c || cell0 < 0 || count < 0 || cell0 + count > c->cells() || (count > 0 && !buf)) return HYG_EINVAL;
    if (c->precision != HYG_F64) return HYG_ENOTSUP;
    if (count == 0) return HYG_OK;
    cudaSetDevice(c->device);
    Layers4 L{{c->s64[c->cur][0], c->s64[c->cur][1], c->s64[c->cur][2], c->s64[c->cur][3]}};
    const int grid = static_cast<int>(std::min<int64_t>((4 * count + 255) / 256, 4 * sm_count(c->device)));
    {
        LaunchScope ls(c, "unpack_cells", 0.0);
        k_unpack_cells<<<grid, 256, 0, c->xstream ? c->xstream : c->stream>>>(L, cell0, count, buf);
    }
    return cudaGetLastError() == cudaSuccess ? HYG_OK : HYG_ECUDA;
}

int hyg_pack_zones(hyg_ctx* c, int32_t z0, int32_t count, double* buf) {
    if (!c || z0 < 0 || count < 0 || z0 + count > static_cast<int>(c->zones.size()) || (count > 0 && !buf))
        return HYG_EINVAL;
    if (count == 0) return HYG_OK;
    cudaSetDevice(c->device);
    cudaStream_t xs = c->xstream ? c->xstream : c->stream;
    if (cudaMemcpyAsync(buf, c->zu[c->zcur] + z0, count * sizeof(double), cudaMemcpyDeviceToDevice, xs) ||
        cudaMemcpyAsync(buf + count, c->zv[c->zcur] + z0, count * sizeof(double), cudaMemcpyDeviceToDevice, xs))
        return HYG_ECUDA;
    return HYG_OK;
}

int hyg_unpack_zones(hyg_ctx* c, int32_t z0, int32_t count, const double* buf) {
    if (!c || z0 < 0 || count < 0 || z0 + count > static_cast<int>(c->zones.size()) || (count > 0 && !buf))
        return HYG_EINVAL;
    if (count == 0) return HYG_OK;
    cudaSetDevice(c->device);
    cudaStream_t xs = c->xstream ? c->xstream : c->stream;
    if (cudaMemcpyAsync(c->zu[c->zcur] + z0, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, xs) ||
        cudaMemcpyAsync(c->zv[c->zcur] + z0, buf + count, count * sizeof(double), cudaMemcpyDeviceToDevice, xs))
        return HYG_ECUDA;
    return HYG_OK;
}

int hyg_set_tuning(hyg_ctx* c, int32_t knob, int64_t value) {
    if (!c || value < 0) return HYG_EINVAL;
    switch (knob) {
        case HYG_TUNE_RING_GRID: c->ring_grid_cap = static_cast<int>(std::min<int64_t>(value, INT32_MAX)); return HYG_OK;
        case HYG_TUNE_RING_KERNEL:
            if (value > 4) return HYG_EINVAL;
            c->ring_kernel = static_cast<int>(value);
            return HYG_OK;
        case HYG_TUNE_RING_DEPTH:
            if (value < 1 || value > kRingSplitMaxM) return HYG_EINVAL;
            c->ring_split_m = static_cast<int>(value);
            return HYG_OK;
        case HYG_TUNE_TILED_LOAD:
            if (value > 1) return HYG_EINVAL;
            c->tiled_load = static_cast<int>(value);
            return HYG_OK;
        case HYG_TUNE_MATERIAL_EXACT:
            if (value > 1) return HYG_EINVAL;
            c->mat_exact = value != 0;
            return HYG_OK;
        default: return HYG_EINVAL;
    }
}

int hyg_reset_kernel_stats(hyg_ctx* c) {
    if (!c) return HYG_EINVAL;
    hyg_synchronize(c);
    c->stats.clear();
    return HYG_OK;
}
int64_t hyg_launch_count(hyg_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"

// ---- FP64 pipe probe (roofline denominator; MEASURED_PEAKS.json has no FP64) ----
namespace {
__global__ void k_dfma_probe(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
}  // namespace

namespace {
__global__ void k_ffma_probe(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-6f + k;
    const float b = 0.9999f, c = 1e-4f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

namespace {
__global__ void k_fastmath(int n, const double* x, double* e, double* r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        e[i] = fexp(x[i], kExp2Tab64);
        r[i] = frcp(x[i]);
    }
}
// the d(v) half node's exp (-700 <= x <= 0) and the v row's two-FMA reciprocal
__global__ void k_dvmath(int n, const double* x, double* e, double* r) {
    __shared__ double s_tab[256];
    for (int j = threadIdx.x; j < 256; j += blockDim.x) s_tab[j] = exp_tab_biased(j);
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        e[i] = fexp_addend<1>(-fabs(x[i]), s_tab);
        r[i] = frcp2(x[i]);
    }
}
// df_step_linear (wall.cpp:60-71) of n_fields independent single fields:
// next[j] = a0 prev[j] + a1 (curr[j+1] + curr[j-1]) inside, ends copied
__global__ void k_df_linear(int n_fields, int n, double a0, double a1, const double* prev, const double* curr,
                            double* next) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n_fields) * n) return;
    const int j = static_cast<int>(i % n);
    next[i] = (j == 0 || j == n - 1) ? curr[i] : a0 * prev[i] + a1 * (curr[i + 1] + curr[i - 1]);
}

__global__ void k_crmath(int n, const double* x, const double* y, double* o) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        o[i] = cr::exp(x[i]);
        o[n + i] = cr::log(x[i]);
        o[2 * n + i] = cr::log10(x[i]);
        o[3 * n + i] = cr::pow(x[i], y[i]);
    }
}
__global__ void k_fastlog(int n, const double* x, double* l) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) l[i] = flog_pos(x[i]);
}
}  // namespace

extern "C" int hyg_df_march_linear(int32_t device, int32_t n_fields, int32_t n, double lambda, int64_t steps,
                                   double* prev, double* curr) {
    hyg_status* status = nullptr;
    if (n_fields < 0 || n < 2 || steps < 0 || !prev || !curr) return HYG_EINVAL;
    if (n_fields == 0 || steps == 0) return HYG_OK;
    HYG_CUDA(cudaSetDevice(device));
    const size_t cells = static_cast<size_t>(n_fields) * n, bytes = cells * sizeof(double);
    double* d = nullptr;
    HYG_CUDA(cudaMalloc(&d, 3 * bytes));
    double* L[3] = {d, d + cells, d + 2 * cells};
    HYG_CUDA(cudaMemcpy(L[0], prev, bytes, cudaMemcpyDefault));
    HYG_CUDA(cudaMemcpy(L[1], curr, bytes, cudaMemcpyDefault));
    const double a0 = (1.0 - lambda) / (1.0 + lambda);   // wall.cpp:66-67
    const double a1 = lambda / (1.0 + lambda);
    const int grid = static_cast<int>((cells + 255) / 256);
    for (int64_t k = 0; k < steps; ++k) {                // rotate (wall.cpp:80-83) by renaming
        k_df_linear<<<grid, 256>>>(n_fields, n, a0, a1, L[0], L[1], L[2]);
        double* t = L[0];
        L[0] = L[1];
        L[1] = L[2];
        L[2] = t;
    }
    HYG_CUDA(cudaGetLastError());
    HYG_CUDA(cudaMemcpy(prev, L[0], bytes, cudaMemcpyDefault));
    HYG_CUDA(cudaMemcpy(curr, L[1], bytes, cudaMemcpyDefault));
    cudaFree(d);
    return HYG_OK;
}

extern "C" int hyg_selftest_crmath(int32_t device, int32_t n, const double* x, const double* y, double* out) {
    hyg_status* status = nullptr;
    if (n <= 0 || !x || !y || !out) return HYG_EINVAL;
    HYG_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    HYG_CUDA(cudaMalloc(&d, sizeof(double) * 6 * n));
    HYG_CUDA(cudaMemcpy(d, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    HYG_CUDA(cudaMemcpy(d + n, y, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_crmath<<<(n + 255) / 256, 256>>>(n, d, d + n, d + 2 * n);
    HYG_CUDA(cudaGetLastError());
    HYG_CUDA(cudaMemcpy(out, d + 2 * n, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return HYG_OK;
}

extern "C" int hyg_selftest_fastlog(int32_t device, int32_t n, const double* x, double* log_out) {
    hyg_status* status = nullptr;
    if (n <= 0 || !x || !log_out) return HYG_EINVAL;
    HYG_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    HYG_CUDA(cudaMalloc(&d, sizeof(double) * 2 * n));
    HYG_CUDA(cudaMemcpy(d, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_fastlog<<<(n + 255) / 256, 256>>>(n, d, d + n);
    HYG_CUDA(cudaGetLastError());
    HYG_CUDA(cudaMemcpy(log_out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return HYG_OK;
}

extern "C" int hyg_selftest_fastmath(int32_t device, int32_t n, const double* x, double* exp_out,
                                     double* rcp_out) {
    hyg_status* status = nullptr;
    if (n <= 0 || !x || !exp_out || !rcp_out) return HYG_EINVAL;
    HYG_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    HYG_CUDA(cudaMalloc(&d, sizeof(double) * 3 * n));
    HYG_CUDA(cudaMemcpy(d, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_fastmath<<<(n + 255) / 256, 256>>>(n, d, d + n, d + 2 * n);
    HYG_CUDA(cudaGetLastError());
    HYG_CUDA(cudaMemcpy(exp_out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
    HYG_CUDA(cudaMemcpy(rcp_out, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return HYG_OK;
}

extern "C" int hyg_selftest_dvmath(int32_t device, int32_t n, const double* x, double* exp_out, double* rcp_out) {
    hyg_status* status = nullptr;
    if (n <= 0 || !x || !exp_out || !rcp_out) return HYG_EINVAL;
    HYG_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    HYG_CUDA(cudaMalloc(&d, sizeof(double) * 3 * n));
    HYG_CUDA(cudaMemcpy(d, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_dvmath<<<(n + 255) / 256, 256>>>(n, d, d + n, d + 2 * n);
    HYG_CUDA(cudaGetLastError());
    HYG_CUDA(cudaMemcpy(exp_out, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
    HYG_CUDA(cudaMemcpy(rcp_out, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return HYG_OK;
}

extern "C" int hyg_probe_fp32_peak(int32_t device, double* tflops) {
    hyg_status* status = nullptr;
    HYG_CUDA(cudaSetDevice(device));
    int sms = 0;
    HYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = sms * 8, threads = 256, iters = 40000;
    float* o = nullptr;
    HYG_CUDA(cudaMalloc(&o, sizeof(float) * blocks * threads));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_ffma_probe<<<blocks, threads>>>(o, 200);
    cudaEventRecord(e0);
    k_ffma_probe<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    HYG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(o);
    if (tflops) *tflops = 2.0 * 64.0 * iters * static_cast<double>(blocks) * threads / (ms * 1e-3) / 1e12;
    return HYG_OK;
}

extern "C" int hyg_probe_fp64_peak(int32_t device, double* tflops, double* sm_clock_mhz) {
    hyg_status* status = nullptr;
    HYG_CUDA(cudaSetDevice(device));
    int sms = 0, clk = 0;
    HYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    double* o = nullptr;
    HYG_CUDA(cudaMalloc(&o, sizeof(double) * blocks * threads));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma_probe<<<blocks, threads>>>(o, 200);   // warm-up
    cudaEventRecord(e0);
    k_dfma_probe<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    HYG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(o);
    const double flops = 2.0 * 64.0 * iters * static_cast<double>(blocks) * threads;
    if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
    if (sm_clock_mhz) *sm_clock_mhz = clk / 1000.0;
    return HYG_OK;
}

#if RING_PROF
// timing variants only (tools/_ringvar): the K4r phase stamps of CTA 0
extern "C" int hyg_ring_prof_read(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_ring_prof, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 5;
}
#endif
