// psdf.cu — host side of the C ABI declared in include/psdf.h.
//
// One context per GPU.  Device state (SoA fp32):
//   params  = [raw T*4096 | planes T*3*256*n_s | probes P*l^2*n_a | mlp]
//   smooth  = [T*4096]                     (SparseGrid smoothed SDF)
//   grads   = same layout as params        (GradBuffers minus staging)
//   gsmooth = [T*4096]                     (smooth-staged SDF gradient)
//   adam m, v = same layout as params
//   tile_table [nt0*nt1*nt2] int32, probe_table [(nt0+1)(nt1+1)(nt2+1)] int32
// A train step: sat_dist -> K2 (the ray pass, psdf_train.cuh) with K3..K6
// (regularizers) and the empty rays' photo terms on a low-priority side
// stream -> K7 (G^T fold) -> [NCCL all-reduce] -> K8 (Adam) -> K9 (smoothing
// + apron); one host synchronisation at the end (buffer overflow -> redo).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>
#include <unordered_set>

#include "../../include/psdf.h"
#include "psdf_grid.cuh"
#include "psdf_raypass.cuh"
#include "psdf_train.cuh"
#include "psdf_lod.cuh"
#include "psdf_mesh.cuh"

using namespace psdf;

namespace {

thread_local std::string g_err;

struct Failure {
    int code;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    throw Failure{code};
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) fail(PSDF_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                    __FILE__, __LINE__);                                       \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return PSDF_OK;
    } catch (const Failure& e) {
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PSDF_ERR_RUNTIME;
    }
}

// ------------------------------------------------------------------ NCCL
struct Nccl {
    void* so = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    void load() {
        if (so) return;
        // NCCL is loaded lazily so single-GPU use has no NCCL dependency; the
        // process-wide libnccl.so.2 (e.g. torch's) is reused when present.
        so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!so) fail(PSDF_ERR_NCCL, "cannot load libnccl.so.2: %s", dlerror());
        GetUniqueId = (decltype(GetUniqueId))dlsym(so, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(so, "ncclCommInitRank");
        AllReduce = (decltype(AllReduce))dlsym(so, "ncclAllReduce");
        ReduceScatter = (decltype(ReduceScatter))dlsym(so, "ncclReduceScatter");
        AllGather = (decltype(AllGather))dlsym(so, "ncclAllGather");
        CommDestroy = (decltype(CommDestroy))dlsym(so, "ncclCommDestroy");
        GetErrorString = (decltype(GetErrorString))dlsym(so, "ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !AllReduce || !ReduceScatter || !AllGather || !CommDestroy ||
            !GetErrorString)
            fail(PSDF_ERR_NCCL, "libnccl.so.2 lacks the expected symbols");
    }
};
Nccl g_nccl;

#define NK(x)                                                                              \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) fail(PSDF_ERR_NCCL, "%s: %s", #x, g_nccl.GetErrorString(r_)); \
    } while (0)

struct DevView {
    psdf_camera cam;
    float* rgb = nullptr;
    uint8_t* mask = nullptr;
};

// Gaussian taps of grid.cpp:10-22, evaluated in f64.
Taps gaussian_taps() {
    double w[5], sum = 0.0;
    for (int d = -2; d <= 2; ++d) {
        w[d + 2] = std::exp(-0.5 * d * d);
        sum += w[d + 2];
    }
    Taps t;
    for (int i = 0; i < 5; ++i) t.w[i] = (float)(w[i] / sum);
    return t;
}

bool supported_channels(int ns, int na) {
#ifdef PSDF_DEV_MINIMAL
    return (ns == 2 && na == 2) || (ns == 4 && na == 4);
#endif
    return (ns == 2 && na == 2) || (ns == 4 && na == 4) || (ns == 8 && na == 8) ||
           (ns == 4 && na == 8) || (ns == 8 && na == 4);
}

// Kernel widths for a caller's (n_s, n_a): the instantiated pair itself, or
// the smallest instantiated pair that holds it.  The extra channels are zero
// planes / probes with zero W1 columns, which leaves every result unchanged:
// the MLP input gains 0 * 0 terms, the feature and probe gradients of a zero
// W1 column are zero, so Adam keeps them at zero, and the feature / probe
// regularizers (losses.cpp:222-290) are plain sums whose zero channels add 0.
bool kernel_widths(int ns, int na, int* ks, int* ka) {
    if (supported_channels(ns, na)) {
        *ks = ns;
        *ka = na;
        return true;
    }
    if (ns < 1 || na < 1) return false;
    static const int pairs[5][2] = {{2, 2}, {4, 4}, {4, 8}, {8, 4}, {8, 8}};
    for (const auto& q : pairs)
        if (q[0] >= ns && q[1] >= na && supported_channels(q[0], q[1])) {
            *ks = q[0];
            *ka = q[1];
            return true;
        }
    return false;
}

// Row-wise repack of a [rows][ws] array into [rows][wd] (zero fill / strip).
void repack_rows(const float* src, int64_t rows, int ws, float* dst, int wd) {
    const int w = std::min(ws, wd);
    for (int64_t r = 0; r < rows; ++r) {
        std::copy(src + r * ws, src + r * ws + w, dst + r * wd);
        std::fill(dst + r * wd + w, dst + (r + 1) * wd, 0.f);
    }
}

// DecoderMlp blob (decoder.hpp:17-31, W1 [32][n_s + n_a + 6] first) between
// the caller's widths (s0, a0) and (s1, a1): W1 columns re-indexed per input
// group (spatial, angular, Fresnel powers), columns of padded channels zero,
// everything after W1 copied.
void repack_mlp(const float* src, int s0, int a0, float* dst, int s1, int a1, int ncam) {
    const int in0 = s0 + a0 + NPOW, in1 = s1 + a1 + NPOW;
    for (int j = 0; j < HID; ++j) {
        float* row = dst + (int64_t)j * in1;
        std::fill(row, row + in1, 0.f);
        const float* r0 = src + (int64_t)j * in0;
        for (int i = 0; i < std::min(s0, s1); ++i) row[i] = r0[i];
        for (int i = 0; i < std::min(a0, a1); ++i) row[s1 + i] = r0[s0 + i];
        for (int i = 0; i < NPOW; ++i) row[s1 + a1 + i] = r0[s0 + a0 + i];
    }
    const MlpLayout L0 = MlpLayout::make(in0), L1 = MlpLayout::make(in1);
    const int64_t tail = (int64_t)L0.cam + (int64_t)ncam * HID - L0.b1;
    std::copy(src + L0.b1, src + L0.b1 + tail, dst + L1.b1);
}

template <typename F>
void dispatch_channels(int ns, int na, F&& f) {
    if (ns == 2 && na == 2) f.template operator()<2, 2>();
    else if (ns == 4 && na == 4) f.template operator()<4, 4>();
#ifndef PSDF_DEV_MINIMAL
    else if (ns == 8 && na == 8) f.template operator()<8, 8>();
    else if (ns == 4 && na == 8) f.template operator()<4, 8>();
    else if (ns == 8 && na == 4) f.template operator()<8, 4>();
#endif
    else fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported (n_s, n_a) = (%d, %d)", ns, na);
}

template <class F>
void dispatch_ns(int ns, F&& f) {
    if (ns == 2) f.template operator()<2>();
    else if (ns == 4) f.template operator()<4>();
    else if (ns == 8) f.template operator()<8>();
    else fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported n_s = %d", ns);
}

int64_t up4(int64_t x) { return (x + 3) & ~int64_t(3); }

// K2a round 0 steps before the remaining rays continue, compacted, in round 1.
constexpr int kComposite0Steps = 16;  // default; PSDF_COMPOSITE_STEPS overrides (tuning)

// Zero floats after the flat parameter / gradient / moment vectors: the
// sharded exchange splits them into world-size chunks of a multiple of 4
// floats (<= n_params + 4 * world).
constexpr int64_t kParamPad = 4096;

// Tile bitmaps up to 32 KB (1024^3 grids) are staged in shared memory.
constexpr int kMaxSmemBitWords = 8192;

}  // namespace

struct psdf_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host->device image staging of psdf_train_step
    cudaStream_t side_stream = nullptr;  // low priority: regularizers under the ray pass
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_scanned = nullptr;    // after the composite pass (hand-over bits final, view table written)
    bool fork_regs = false;              // the ray pass records ev_fork (do_train_step)
    bool grads_clear_pending = false;    // gradient clear on the side stream (ev_zeroed)
    cudaEvent_t ev_start = nullptr, ev_zeroed = nullptr;
    bool regs_early = false;             // PSDF_REGS_EARLY: fork the regularizer at step start
    bool fork_after_scan = false;        // PSDF_REGS_AFTER_SCAN: fork it after the scan, not after round 0
    bool regs_serial = false;            // PSDF_REGS_SERIAL: regularizers after the ray pass, main stream
    cudaEvent_t ev_copied = nullptr, ev_copy_free = nullptr;
    bool images_pending = false;           // inside psdf_train_step: the copies may still run
    cudaEvent_t ev_masks = nullptr, ev_rgb = nullptr;  // masks / colours of the step copied
    unsigned* d_hand_bits = nullptr;       // [work tiles] scan hand-over lanes
    float* d_tmin = nullptr;               // [2][work tiles] first / last allocated-tile hit bounds (tile_raster_kernel)
    int64_t tmin_cap = 0;
    int64_t batch_tiles = 0;               // work tiles of the current view table (upload_viewdev)
    int64_t active_tiles = 0;              // work tiles on the scan's list (upload_viewdev)
    int64_t hand_cap = 0;
    cudaEvent_t ev_ray0 = nullptr, ev_ray1 = nullptr, ev_step0 = nullptr, ev_step1 = nullptr;

    // kernels whose dynamic shared-memory limit was raised on this device
    // (function attributes are per CUDA context; a psdf_ctx is used by one
    // host thread at a time)
    std::unordered_set<const void*> attr_done;
    double test_margin = 1e-8;  // PSDF_TEST_MARGIN, read once at creation

    bool has_grid = false;
    psdf_grid_desc desc{};  // device layout: n_s / n_a are the kernel widths
    // the caller's channel widths (the reference's n_s / n_a, any value in
    // [1, 8]); desc holds the instantiated pair they are zero-padded to
    int hns = 0, hna = 0;
    int in_dim = 0;
    int nt[3] = {0, 0, 0};
    int64_t off_raw = 0, off_planes = 0, off_probes = 0, off_mlp = 0, n_params = 0;
    int64_t n_planes = 0, n_probes = 0, mlp_size = 0;
    int32_t* d_tile_table = nullptr;
    uint32_t* d_tile_bits = nullptr;
    uint8_t* d_tile_dist = nullptr;
    int32_t* d_tile_nbr = nullptr; // [T][27] neighbour tile ids
    int occ_tlo[3] = {0, 0, 0}, occ_thi[3] = {-1, -1, -1};  // allocated tiles' bounding box (tile coords)
    uint8_t* d_sat_dist = nullptr; // [T][17^3] per-cell saturation distances of the current ray pass
    // d_sat_dist is a pure function of (d_smooth_ap, tau): kept across ray
    // passes until either changes (every writer of d_smooth_ap clears sat_ok)
    bool sat_ok = false;
    double sat_tau = 0.0;
    int composite_steps = kComposite0Steps;
    bool coop_round1 = true;       // K2a round 1 one warp per ray (PSDF_COOP=0: one lane per ray, A/B)
    bool coop_render = true;       // renders too: round 0 capped, the tail one warp per ray (PSDF_COOP_RENDER=0)
    bool fwd_mma = false;          // K2b decoder MLP on the tensor cores (PSDF_FWD_MMA=1; measured slower, A/B)
    bool stage_fwd = true;         // K2b probe blocks bulk-copied to shared memory (PSDF_STAGE_FWD=0 off)
    int* d_tile_cnt = nullptr;     // [2T] shading records per tile, then their offsets
    void* scan_tmp = nullptr;      // CUB scan storage of the counting sort
    size_t scan_tmp_bytes = 0;
    int tsort_cap = 0;
    int wave_init = 0;             // PSDF_WAVE_INIT: initial ray-pass buffer capacity (tests)
    int bit_words = 0;
    int4* d_tile_coords = nullptr;
    int32_t* d_probe_ids = nullptr;
    int32_t* d_probe_table = nullptr;
    int4* d_probe_coords = nullptr;
    float* d_params = nullptr;
    float* d_smooth = nullptr;
    float* d_smooth_ap = nullptr;  // smoothed SDF with a 1-voxel apron (sampling layout)
    float* d_grads = nullptr;
    float* d_gsmooth = nullptr;
    float* d_grads0 = nullptr;     // stage-0 copies (keep_raypass)
    float* d_gsmooth0 = nullptr;
    float* d_m = nullptr;
    float* d_v = nullptr;
    long adam_t = 0;
    bool keep_raypass = false;

    std::vector<DevView> views;
    float* d_stage_rgb = nullptr;
    uint8_t* d_stage_mask = nullptr;
    size_t stage_px = 0;
    ViewDev* d_viewdev = nullptr;
    int viewdev_cap = 0;
    float* d_render = nullptr;  // render scratch: rgb | alpha | depth
    size_t render_px = 0;
    uint8_t* d_eval = nullptr;  // point-to-mesh scratch (grow-only arena)
    uint8_t* d_mc = nullptr;    // marching-cubes cell arrays + scan storage (grow-only)
    size_t mc_cap = 0;
    uint8_t* d_mesh = nullptr;  // the last extracted mesh: verts f64 | tris i32 (grow-only)
    size_t mesh_cap = 0;
    int64_t mesh_nv = -1, mesh_nt = -1;  // -1: no mesh extracted
    size_t eval_cap = 0;

    unsigned long long* d_work = nullptr;
    unsigned long long* d_counts = nullptr;
    double* d_stats = nullptr;
    double* h_stats = nullptr;              // pinned
    unsigned long long* h_counts = nullptr;  // pinned

    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    int grad_exchange = PSDF_EXCHANGE_ALLREDUCE;  // psdf_set_grad_exchange
    cudaStream_t comm_stream = nullptr;           // bucketed exchange: the [planes|probes|mlp] bucket
    cudaEvent_t ev_bucket = nullptr, ev_bucket_done = nullptr;

    float last_ray_ms = 0.f, last_step_ms = 0.f;
    float last_k2_ms[4] = {0.f, 0.f, 0.f, 0.f};  // K2a, K2b, K2d, K2e
    int last_launches = 0;
    int64_t last_entries = 0, last_records = 0;
    int64_t last_wave[5] = {0, 0, 0, 0, 0};  // entries, records, handovers, continuations, alpha samples
    int64_t last_h2d_bytes = 0;    // host -> device bytes of the last psdf_train_step
    // psdf_train_step: enqueues the colour copies (and records ev_rgb); run
    // once, by the ray pass right after the scan launch (the host scans the
    // masks while the GPU marches) and in any case before the first wait on
    // ev_rgb (run_rgb_copy)
    std::function<void()> rgb_copy;
    // per view [first, last] pixel row holding a mask pixel (mask_rows_kernel
    // on the copy stream, read back into pinned h_rows; ev_rows)
    int* d_rows = nullptr;
    int* h_rows = nullptr;
    int rows_cap = 0;
    cudaEvent_t ev_rows = nullptr;
    cudaEvent_t ev_k[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};

    // wavefront buffers of the train ray pass (psdf_train.cuh)
    WaveBufs wave{};
    unsigned* h_wave_counters = nullptr;  // pinned [8]

    GridView view() const {
        GridView g{};
        g.T = desc.T;
        g.P = desc.P;
        g.n_s = desc.n_s;
        g.n_a = desc.n_a;
        g.order = desc.sh_order;
        for (int a = 0; a < 3; ++a) {
            g.res[a] = desc.res[a];
            g.nt[a] = nt[a];
            g.org[a] = desc.origin[a];
            // world_max() = origin + res * voxel_size (grid.hpp:72-74)
            g.wmax[a] = desc.origin[a] + (double)desc.res[a] * desc.voxel_size;
            g.occ_lo[a] = desc.origin[a] + (double)(occ_tlo[a] * TE - 1) * desc.voxel_size;
            g.occ_hi[a] = desc.origin[a] + (double)((occ_thi[a] + 1) * TE + 1) * desc.voxel_size;
        }
        g.h = desc.voxel_size;
        int ex = 0;
        g.h_pow2 = desc.voxel_size > 0.0 && std::frexp(desc.voxel_size, &ex) == 0.5;
        g.inv_h = g.h_pow2 ? 1.0 / desc.voxel_size : 0.0;
        g.far = desc.far_field_voxels * desc.voxel_size;
        g.occ_any = occ_thi[0] >= occ_tlo[0];
        g.tile_table = d_tile_table;
        g.tile_bits = d_tile_bits;
        g.tile_dist = d_tile_dist;
        g.tile_nbr = d_tile_nbr;
        g.sat_dist = d_sat_dist;
        // decision margin of the marcher's fast paths; PSDF_TEST_MARGIN widens
        // it so the tests drive the exact / rewind paths on most decisions
        g.margin = test_margin;
        g.bit_words = bit_words;
        g.tile_coords = d_tile_coords;
        g.probe_ids = d_probe_ids;
        g.smooth = d_smooth;
        g.smooth_ap = d_smooth_ap;
        g.planes = d_params + off_planes;
        g.probes = d_params + off_probes;
        return g;
    }

    void free_grid() {
        for (void* p : {(void*)d_tile_table, (void*)d_tile_bits, (void*)d_tile_dist, (void*)d_tile_nbr, (void*)d_sat_dist, (void*)d_tile_coords, (void*)d_probe_ids,
                        (void*)d_probe_table, (void*)d_probe_coords, (void*)d_params,
                        (void*)d_smooth, (void*)d_smooth_ap, (void*)d_grads, (void*)d_gsmooth, (void*)d_grads0,
                        (void*)d_gsmooth0, (void*)d_m, (void*)d_v})
            if (p) cudaFree(p);
        d_tile_table = nullptr;
        d_tile_bits = nullptr;
        d_tile_dist = nullptr;
        d_tile_nbr = nullptr;
        d_sat_dist = nullptr;
        d_tile_coords = nullptr;
        d_probe_ids = nullptr;
        d_probe_table = nullptr;
        d_probe_coords = nullptr;
        d_params = d_smooth = d_smooth_ap = d_grads = d_gsmooth = d_grads0 = d_gsmooth0 = d_m = d_v = nullptr;
        has_grid = false;
    }
};

namespace {

void need_grid(psdf_ctx* c) {
    if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
    if (!c->has_grid) fail(PSDF_ERR_RUNTIME, "no grid uploaded");
}

void set_device(psdf_ctx* c) { CK(cudaSetDevice(c->device)); }

template <typename T>
void ensure_dev(T*& p, size_t& cap, size_t n) {
    if (n <= cap && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    cap = n;
}

// Call-scoped device scratch: every buffer is freed when the scope ends,
// including when a failure unwinds it (fail() throws into guarded()).
struct DevScratch {
    std::vector<void*> ptrs;
    DevScratch() = default;
    DevScratch(const DevScratch&) = delete;
    DevScratch& operator=(const DevScratch&) = delete;
    ~DevScratch() { release(); }
    template <typename T>
    T* alloc(size_t n) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    void release() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
    }
};

Cam to_cam(const psdf_camera& c) {
    Cam d;
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    d.rfx = 1.0 / c.fx;  // correctly rounded reciprocals for ddiv_r (psdf_device.cuh)
    d.rfy = 1.0 / c.fy;
    for (int i = 0; i < 9; ++i) d.rot[i] = c.rot[i];
    for (int i = 0; i < 3; ++i) d.pos[i] = c.pos[i];
    d.width = c.width;
    d.height = c.height;
    d.id = c.id;
    return d;
}

void check_camera(const psdf_camera& c) {
    if (c.width <= 0 || c.height <= 0) fail(PSDF_ERR_INVALID_ARGUMENT, "camera has an empty image");
}

// Copies the batch's view table to the device and returns the work-tile count.
// The pixel rectangle of a view whose rays can reach the allocated tiles'
// bounding box (Camera::project of its eight corners, padded by 2 pixels);
// the whole image unless every corner is well in front of the camera.
void occ_rect(const GridView& g, ViewDev& v) {
    const Cam& k = v.cam;
    v.occ_u0 = 0;
    v.occ_u1 = k.width - 1;
    v.occ_v0 = 0;
    v.occ_v1 = k.height - 1;
    if (!g.occ_any) {  // nothing allocated: no ray has a sample
        v.occ_u0 = v.occ_v0 = 1;
        v.occ_u1 = v.occ_v1 = 0;
        return;
    }
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    for (int i = 0; i < 8; ++i) {
        const double p[3] = {(i & 1) ? g.occ_hi[0] : g.occ_lo[0], (i & 2) ? g.occ_hi[1] : g.occ_lo[1],
                             (i & 4) ? g.occ_hi[2] : g.occ_lo[2]};
        const double d[3] = {p[0] - k.pos[0], p[1] - k.pos[1], p[2] - k.pos[2]};
        const double cx = k.rot[0] * d[0] + k.rot[3] * d[1] + k.rot[6] * d[2];
        const double cy = k.rot[1] * d[0] + k.rot[4] * d[1] + k.rot[7] * d[2];
        const double cz = k.rot[2] * d[0] + k.rot[5] * d[1] + k.rot[8] * d[2];
        if (!(cz > 1e-3)) return;  // a corner beside / behind the camera: no culling
        const double u = k.fx * cx / cz + k.cx, w = k.fy * cy / cz + k.cy;
        umin = std::min(umin, u);
        umax = std::max(umax, u);
        vmin = std::min(vmin, w);
        vmax = std::max(vmax, w);
    }
    // pixel u's ray passes through the image point u + 1/2
    auto clampi = [](double x, int lo, int hi) { return (int)std::max<double>(lo, std::min<double>(hi, x)); };
    v.occ_u0 = clampi(std::floor(umin) - 2.0, 0, k.width);
    v.occ_u1 = clampi(std::ceil(umax) + 2.0, -1, k.width - 1);
    v.occ_v0 = clampi(std::floor(vmin) - 2.0, 0, k.height);
    v.occ_v1 = clampi(std::ceil(vmax) + 2.0, -1, k.height - 1);
}

int64_t upload_viewdev(psdf_ctx* c, std::vector<ViewDev>& vd) {
    int64_t tiles = 0, active = 0;
    const GridView g = c->view();
    for (auto& v : vd) {
        v.tiles_x = (v.cam.width + 7) / 8;
        v.tiles_y = (v.cam.height + 3) / 4;
        v.tile_begin = tiles;
        tiles += (int64_t)v.tiles_x * v.tiles_y;
        occ_rect(g, v);
        // work tiles overlapping the occupancy rectangle (the scan's list)
        v.act_begin = active;
        v.act_tx0 = v.act_ty0 = v.act_w = v.act_n = 0;
        if (v.occ_u1 >= v.occ_u0 && v.occ_v1 >= v.occ_v0) {
            v.act_tx0 = v.occ_u0 / 8;
            v.act_ty0 = v.occ_v0 / 4;
            v.act_w = v.occ_u1 / 8 - v.act_tx0 + 1;
            v.act_n = v.act_w * (v.occ_v1 / 4 - v.act_ty0 + 1);
        }
        active += v.act_n;
    }
    c->active_tiles = active;
    c->batch_tiles = tiles;
    if ((int)vd.size() > c->viewdev_cap) {
        if (c->d_viewdev) cudaFree(c->d_viewdev);
        CK(cudaMalloc(&c->d_viewdev, sizeof(ViewDev) * vd.size()));
        c->viewdev_cap = (int)vd.size();
    }
    CK(cudaMemcpyAsync(c->d_viewdev, vd.data(), sizeof(ViewDev) * vd.size(),
                       cudaMemcpyHostToDevice, c->stream));
    return tiles;
}

int camera_bias_row(psdf_ctx* c, int camera_id) {
    if (camera_id < 0 || c->desc.ncam == 0) return -1;  // decoder.cpp:69-78
    if (camera_id >= c->desc.ncam)
        fail(PSDF_ERR_OUT_OF_RANGE, "decode_color: camera id out of range");
    return camera_id;
}

int blocks_per_sm(const void* fn, size_t smem) {
    int n = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, BLOCK, smem));
    return std::max(n, 1);
}

// G^T fold: dst += G * src (src filled with 0 outside allocated tiles).
void launch_fold(psdf_ctx* c, const float* src, float* dst) {
    if (c->desc.T == 0) return;
    if (c->attr_done.insert((const void*)smooth_fold_kernel).second)
        CK(cudaFuncSetAttribute(smooth_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kFoldSmem));
    smooth_fold_kernel<<<c->desc.T, PSDF_FOLD_THREADS, kFoldSmem, c->stream>>>(c->view(), src, 0.f, dst, 1,
                                                                 gaussian_taps());
    CK(cudaGetLastError());
    ++c->last_launches;
}

// Refreshes the apron copy (and brick minima) from the current smoothed grid.
void fill_apron(psdf_ctx* c) {
    if (c->desc.T == 0) return;
    c->sat_ok = false;
    apron_fill_kernel<<<c->desc.T, 256, 0, c->stream>>>(c->view(), c->d_smooth, c->d_smooth_ap);
    CK(cudaGetLastError());
    ++c->last_launches;
}

// SparseGrid::smooth_all (grid.cpp:247-250) + apron + brick minima, one pass.
void smooth_all(psdf_ctx* c) {
    if (c->desc.T == 0) return;
    c->sat_ok = false;
    if (c->attr_done.insert((const void*)smooth_apron_kernel).second)
        CK(cudaFuncSetAttribute(smooth_apron_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kSmoothApronSmem));
    smooth_apron_kernel<<<c->desc.T, PSDF_SMOOTH_THREADS, kSmoothApronSmem, c->stream>>>(
        c->view(), c->d_params + c->off_raw, (float)(c->desc.far_field_voxels * c->desc.voxel_size),
        c->d_smooth, c->d_smooth_ap, gaussian_taps());
    CK(cudaGetLastError());
    ++c->last_launches;
}

// Saturation distances for a ray pass with this tau (the marcher's runs);
// with runs disabled (tau_run <= 0) every block reads as unsaturated.
void prepare_sat(psdf_ctx* c, double tau_run) {
    if (c->desc.T == 0) return;
    if (c->sat_ok && c->sat_tau == tau_run) return;  // same stream: the last pass's table stands
    c->sat_ok = true;
    c->sat_tau = tau_run;
    sat_dist_kernel<<<c->desc.T, kSatThreads, 0, c->stream>>>(c->view(), tau_run, c->d_sat_dist);
    CK(cudaGetLastError());
    ++c->last_launches;
}



void free_wave(psdf_ctx* c) {
    WaveBufs& W = c->wave;
    for (void* p : {(void*)W.e_slot, (void*)W.e_dir, (void*)W.e_tfirst, (void*)W.e_cfirst,
                    (void*)W.e_nlive, (void*)W.e_acc, (void*)W.e_head, (void*)W.e_craw, (void*)W.e_t1,
                    (void*)W.r_pos, (void*)W.r_w, (void*)W.r_tile, (void*)W.r_entry,
                    (void*)W.r_next, (void*)W.r_c, (void*)W.r_up, (void*)W.r_geo, (void*)W.h_slot,
                    (void*)W.h_count, (void*)W.h_tileprev, (void*)W.h_t, (void*)W.h_tprev, (void*)W.h_dir,
                    (void*)W.h_t1, (void*)W.r_perm, (void*)W.r_fg, (void*)W.k_rec, (void*)W.a_t,
                    (void*)W.a_s, (void*)W.a_i, (void*)W.e_ahead})
        if (p) cudaFree(p);
    unsigned* keep = W.counters;
    W = WaveBufs{};
    W.counters = keep;
}

// Grows the ray-pass buffers (kept across steps).
void ensure_wave(psdf_ctx* c, int64_t e_cap, int64_t r_cap, int64_t h_cap, int64_t k_cap, int64_t a_cap) {
    WaveBufs& W = c->wave;
    if (e_cap <= W.e_cap && r_cap <= W.r_cap && h_cap <= W.h_cap && k_cap <= W.k_cap && a_cap <= W.a_cap) return;
    e_cap = std::max<int64_t>(e_cap, W.e_cap);
    r_cap = std::max<int64_t>(r_cap, W.r_cap);
    h_cap = std::max<int64_t>(h_cap, W.h_cap);
    k_cap = std::max<int64_t>(k_cap, W.k_cap);
    a_cap = std::max<int64_t>(a_cap, W.a_cap);
    if (e_cap > INT32_MAX / 4 || r_cap > INT32_MAX / 4 || h_cap > INT32_MAX / 4 || a_cap > INT32_MAX / 4)
        fail(PSDF_ERR_RUNTIME, "ray pass needs more than 2^29 entries / records");
    CK(cudaStreamSynchronize(c->stream));
    free_wave(c);
    CK(cudaMalloc(&W.e_slot, sizeof(int) * e_cap));
    CK(cudaMalloc(&W.e_dir, sizeof(double) * 3 * e_cap));
    CK(cudaMalloc(&W.e_tfirst, sizeof(double) * e_cap));
    CK(cudaMalloc(&W.e_cfirst, sizeof(int) * e_cap));
    CK(cudaMalloc(&W.e_nlive, sizeof(int) * e_cap));
    CK(cudaMalloc(&W.e_acc, sizeof(double) * e_cap));
    CK(cudaMalloc(&W.e_head, sizeof(int) * e_cap));
    CK(cudaMalloc(&W.e_craw, sizeof(double) * 3 * e_cap));
    CK(cudaMalloc(&W.e_t1, sizeof(double) * e_cap));
    CK(cudaMalloc(&W.e_ahead, sizeof(int) * e_cap));
    CK(cudaMalloc(&W.r_pos, sizeof(double) * 3 * r_cap));
    CK(cudaMalloc(&W.r_w, sizeof(double) * r_cap));
    CK(cudaMalloc(&W.r_tile, sizeof(int) * r_cap));
    CK(cudaMalloc(&W.r_entry, sizeof(int) * r_cap));
    CK(cudaMalloc(&W.r_next, sizeof(int) * r_cap));
    CK(cudaMalloc(&W.r_c, sizeof(float4) * r_cap));
    CK(cudaMalloc(&W.r_up, sizeof(float4) * r_cap));
    // geometry records sized for the widest supported channel configuration
    CK(cudaMalloc(&W.r_geo, sizeof(float) * (size_t)GeoRec<8, 8>::STRIDE * r_cap));
    CK(cudaMalloc(&W.r_perm, sizeof(int) * r_cap));
    CK(cudaMalloc(&W.r_fg, sizeof(float) * (size_t)FgDims<8, 8>::STRIDE * r_cap));
    CK(cudaMalloc(&W.h_slot, sizeof(int) * h_cap));
    CK(cudaMalloc(&W.h_count, sizeof(int) * h_cap));
    CK(cudaMalloc(&W.h_tileprev, sizeof(int) * h_cap));
    CK(cudaMalloc(&W.h_t, sizeof(double) * h_cap));
    CK(cudaMalloc(&W.h_tprev, sizeof(double) * h_cap));
    CK(cudaMalloc(&W.h_dir, sizeof(double) * 3 * h_cap));
    CK(cudaMalloc(&W.h_t1, sizeof(double) * h_cap));
    CK(cudaMalloc(&W.k_rec, sizeof(ContRec) * k_cap));
    CK(cudaMalloc(&W.a_t, sizeof(double) * 2 * a_cap));
    CK(cudaMalloc(&W.a_s, sizeof(double) * 3 * a_cap));
    CK(cudaMalloc(&W.a_i, sizeof(int4) * a_cap));
    W.e_cap = (int)e_cap;
    W.r_cap = (int)r_cap;
    W.h_cap = (int)h_cap;
    W.k_cap = (int)k_cap;
    W.a_cap = (int)a_cap;
}

// Per-tile record counts / offsets of the counting sort, and its scan storage.
void ensure_tile_sort(psdf_ctx* c) {
    const int T = c->desc.T;
    if (T <= c->tsort_cap) return;
    CK(cudaStreamSynchronize(c->stream));
    if (c->d_tile_cnt) cudaFree(c->d_tile_cnt);
    if (c->scan_tmp) cudaFree(c->scan_tmp);
    c->d_tile_cnt = nullptr;
    c->scan_tmp = nullptr;
    CK(cudaMalloc(&c->d_tile_cnt, sizeof(int) * 2 * (size_t)T));
    c->scan_tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, c->scan_tmp_bytes, c->d_tile_cnt, c->d_tile_cnt + T, T, c->stream));
    CK(cudaMalloc(&c->scan_tmp, std::max<size_t>(c->scan_tmp_bytes, 16)));
    c->tsort_cap = T;
}

// After the step's final synchronisation: true (and larger buffers) when the
// ray pass overflowed one of them; the caller redoes the pass.
bool wave_overflowed(psdf_ctx* c) {
    const unsigned* h = c->h_wave_counters;
    const WaveBufs& W = c->wave;
    if (h[0] <= (unsigned)W.e_cap && h[1] <= (unsigned)W.r_cap && h[2] <= (unsigned)W.h_cap &&
        h[3] <= (unsigned)W.k_cap && h[4] <= (unsigned)W.a_cap)
        return false;
    auto grow = [](unsigned n) { return (int64_t)n + n / 2 + 4096; };
    ensure_wave(c, grow(h[0]), grow(h[1]), grow(h[2]), grow(h[3]), grow(h[4]));
    return true;
}

// K2 as the wavefront pipeline K2a-scan -> K2a (two rounds) -> [records by
// tile] -> K2b -> K2d -> K2e (psdf_train.cuh), with no host round trip: the
// kernels read their item counts on device, the counters are copied back with
// the step's results (wave_overflowed() checks them).
// First / last row in [r0, r1] of a mask with a nonzero byte (warp per row):
// rows[0] atomicMin as unsigned, rows[1] atomicMax (both preset to -1).
__global__ void __launch_bounds__(256) mask_rows_kernel(const uint8_t* __restrict__ mask, int w, int r0, int r1,
                                                        int* __restrict__ rows) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int r = r0 + blockIdx.x * wpb + (threadIdx.x >> 5); r <= r1; r += gridDim.x * wpb) {
        const uint8_t* q = mask + (size_t)r * w;
        bool any = false;
        for (int k = lane; k < w; k += 32) any |= q[k] != 0;
        if (__any_sync(0xffffffffu, any) && lane == 0) {
            atomicMin(reinterpret_cast<unsigned*>(rows), (unsigned)r);
            atomicMax(rows + 1, r);
        }
    }
}

// The deferred colour copies of psdf_train_step (no-op once done / for
// resident images).  Every wait on ev_rgb is preceded by this call.
bool run_rgb_copy(psdf_ctx* c) {
    if (!c->rgb_copy) return false;
    std::function<void()> f = std::move(c->rgb_copy);
    c->rgb_copy = nullptr;
    f();
    return true;
}

template <int NS, int NA>
void launch_train_raypass(psdf_ctx* c, RayPassParams& P, int64_t n_rays) {
    cudaStream_t s = c->stream;
    const int64_t n_work = P.tile_end - P.tile_begin;
    if (c->wave.e_cap == 0) {
        if (c->wave_init > 0)  // tests: force the overflow / redo path
            ensure_wave(c, c->wave_init, c->wave_init, c->wave_init, c->wave_init, c->wave_init);
        else
            ensure_wave(c, n_rays / 8 + 65536, n_rays / 8 + 65536, n_rays / 2 + 65536, n_rays / 16 + 65536,
                        n_rays / 8 + 65536);
    }
    ensure_tile_sort(c);
    const size_t smem_f = render_smem_bytes<NS, NA>();
    const size_t smem_b = shade_bwd_smem_bytes<NS, NA>();
    const size_t smem_fm = shade_fwd_mma_smem_bytes<NS, NA>();
    const size_t smem_bits = sizeof(uint32_t) * P.bits_sm_words;
    if (c->attr_done.insert((const void*)shade_fwd_kernel<NS, NA, true>).second) {
        CK(cudaFuncSetAttribute(shade_fwd_kernel<NS, NA, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f));
        CK(cudaFuncSetAttribute(shade_fwd_kernel<NS, NA, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f));
        CK(cudaFuncSetAttribute(shade_fwd_mma_kernel<NS, NA, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fm));
        CK(cudaFuncSetAttribute(shade_fwd_mma_kernel<NS, NA, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fm));
        CK(cudaFuncSetAttribute(shade_bwd_kernel<NS, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b));
        CK(cudaFuncSetAttribute(march_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(uint32_t) * kMaxSmemBitWords)));
        CK(cudaFuncSetAttribute(march_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(uint32_t) * kMaxSmemBitWords)));
        CK(cudaFuncSetAttribute(march_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(uint32_t) * kMaxSmemBitWords)));
    }
    const int per_sm_s = blocks_per_sm((const void*)march_scan_kernel, smem_bits);
    const int64_t grid_s = std::max<int64_t>(1, std::min<int64_t>((n_work + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK,
                                                                   (int64_t)per_sm_s * c->sm_count));
    const int grid_a = blocks_per_sm((const void*)march_fwd_kernel, smem_bits) * c->sm_count;
    const int grid_c1 = blocks_per_sm((const void*)march_coop_kernel, smem_bits) * c->sm_count;
    WaveBufs W = c->wave;
    CK(cudaEventRecord(c->ev_ray0, s));
    CK(cudaEventRecord(c->ev_k[0], s));
    CK(cudaMemsetAsync(c->d_work, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(W.counters, 0, sizeof(unsigned) * 8, s));
    P.work_counter = c->d_work;
    if (c->hand_cap < n_work) {  // per work tile: which lanes the scan handed over
        if (c->d_hand_bits) cudaFree(c->d_hand_bits);
        c->d_hand_bits = nullptr;
        CK(cudaMalloc(&c->d_hand_bits, sizeof(unsigned) * std::max<int64_t>(n_work, 1)));
        c->hand_cap = n_work;
    }
    c->wave.hand_bits = W.hand_bits = c->d_hand_bits;
    // the scan reads no image: with psdf_train_step it runs under the copies
    // the scan visits only the active work tiles; the others keep hand-over
    // bits 0 (train: empty-ray terms) / the background (render: filled here)
    P.scan_lo = 0;
    P.scan_hi = c->active_tiles;
    // per work tile: lower bound on the first allocated-tile hit (tile_raster_kernel)
    const int64_t all_tiles = c->batch_tiles;  // every view's work tiles (this rank scans its slice)
    if (c->tmin_cap < all_tiles) {
        if (c->d_tmin) cudaFree(c->d_tmin);
        c->d_tmin = nullptr;
        CK(cudaMalloc(&c->d_tmin, 2 * sizeof(float) * std::max<int64_t>(all_tiles, 1)));
        c->tmin_cap = all_tiles;
    }
    {
        const int64_t nt = std::max<int64_t>(all_tiles, 1);
        CK(cudaMemsetAsync(c->d_tmin, 0x7F, sizeof(float) * nt, s));
        CK(cudaMemsetAsync(c->d_tmin + c->tmin_cap, 0, sizeof(float) * nt, s));
        const int64_t warps = (int64_t)c->desc.T * P.n_views;
        if (warps > 0) {
            tile_raster_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(P.g, P.views, P.n_views, c->d_tmin,
                                                                          c->d_tmin + c->tmin_cap);
            CK(cudaGetLastError());
            ++c->last_launches;
        }
    }
    P.tile_tmin = c->d_tmin;
    P.tile_tmax = c->d_tmin + c->tmin_cap;
    if (P.mode != 1) {
        CK(cudaMemsetAsync(W.hand_bits, 0, sizeof(unsigned) * std::max<int64_t>(n_work, 1), s));
    } else {
        render_fill_kernel<<<4 * c->sm_count, 256, 0, s>>>(P, n_work);
        CK(cudaGetLastError());
        ++c->last_launches;
    }
    march_scan_kernel<<<(unsigned)grid_s, BLOCK, smem_bits, s>>>(P, W);
    CK(cudaGetLastError());
    ++c->last_launches;
    // handovers in append order: a warp's handovers come from one 8x4 pixel
    // tile and neighbouring warps from neighbouring work tiles (a sort by
    // pixel measured slower than it saved)
    CK(cudaMemsetAsync(c->d_work, 0, sizeof(unsigned long long), s));
    if (c->fork_regs && c->fork_after_scan) CK(cudaEventRecord(c->ev_fork, s));
    // the composite pass reads the masks (which rays are shaded)
    if (c->images_pending) CK(cudaStreamWaitEvent(s, c->ev_masks, 0));
    // round 0 one lane per ray for `composite_steps` steps, then the rays
    // still alive one warp per ray (march_coop_kernel); PSDF_COOP=0 keeps
    // one lane per ray (a render then runs one uncapped round)
    const bool coop = c->coop_round1 && (P.mode != 1 || c->coop_render);
    march_fwd_kernel<<<(unsigned)grid_a, BLOCK, smem_bits, s>>>(P, W, 0, P.mode == 1 && !coop ? INT_MAX : c->composite_steps);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(c->d_work, 0, sizeof(unsigned long long), s));
    if (c->fork_regs && !c->fork_after_scan) CK(cudaEventRecord(c->ev_fork, s));
    if (coop)
        march_coop_kernel<<<(unsigned)grid_c1, BLOCK, smem_bits, s>>>(P, W);
    else
        march_fwd_kernel<<<(unsigned)grid_a, BLOCK, smem_bits, s>>>(P, W, 1, INT_MAX);
    CK(cudaGetLastError());
    // the empty rays' photo terms (side stream) read the hand-over bits (the
    // scan's, less the rays the composite pass ended without an alpha > 0
    // settle) and the view table: they wait for this point
    CK(cudaEventRecord(c->ev_scanned, s));
    c->last_launches += 2;
    if (getenv("PSDF_DEBUG_MARCH")) {
        unsigned long long cc[8];
        unsigned hw[8];
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpy(cc, c->d_counts, sizeof cc, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hw, W.counters, sizeof hw, cudaMemcpyDeviceToHost));
        fprintf(stderr, "[psdf] march exact fallbacks: %llu; handovers %u entries %u records %u continuations %u "
                "alpha samples %u\n", cc[6], hw[2], hw[0], hw[1], hw[3], hw[4]);
#ifdef PSDF_MARCH_STATS
        unsigned long long st[12];
        CK(cudaMemcpyFromSymbol(st, g_march_stats, sizeof st));
        const unsigned long long zero[12] = {};
        CK(cudaMemcpyToSymbol(g_march_stats, zero, sizeof zero));
        fprintf(stderr, "[psdf] march stats: rays %llu in-box %llu iters %llu samples %llu jumps %llu "
                "skips %llu exact %llu rewinds %llu sat-runs %llu run-samples %llu | probe groups %llu members %llu\n", st[0], st[1], st[2], st[3], st[4], st[5], st[6], st[7], st[8], st[9], st[10], st[11]);
        unsigned long long hh[2][16];
        CK(cudaMemcpyFromSymbol(hh, g_cont_hist, sizeof hh));
        const unsigned long long z2[2][16] = {};
        CK(cudaMemcpyToSymbol(g_cont_hist, z2, sizeof z2));
        unsigned long long cs[8];
        CK(cudaMemcpyFromSymbol(cs, g_coop_stats, sizeof cs));
        CK(cudaMemcpyToSymbol(g_coop_stats, zero, sizeof cs));
        fprintf(stderr, "[psdf] coop: rays %llu steps %llu sat-runs %llu batches %llu batch-samples %llu "
                "single-sample batches %llu\n", cs[0], cs[1], cs[2], cs[3], cs[4], cs[5]);
        for (int r = 0; r < 2; ++r) {
            fprintf(stderr, "[psdf] K2a round %d rays by steps [2^(b-1), 2^b):", r);
            for (int b = 0; b < 16; ++b) fprintf(stderr, " %llu", hh[r][b]);
            fprintf(stderr, "\n");
        }
#endif
    }
    // shading records grouped by tile (K2b / K2e order)
    const int T = c->desc.T;
    const int grid_c = 4 * c->sm_count;
    CK(cudaMemsetAsync(c->d_tile_cnt, 0, sizeof(int) * T, s));
    rec_tile_count_kernel<<<grid_c, 256, 0, s>>>(W, c->d_tile_cnt);
    CK(cudaGetLastError());
    CK(cub::DeviceScan::ExclusiveSum(c->scan_tmp, c->scan_tmp_bytes, c->d_tile_cnt, c->d_tile_cnt + T, T, s));
    rec_tile_scatter_kernel<<<grid_c, 256, 0, s>>>(W, c->d_tile_cnt + T);
    CK(cudaGetLastError());
    c->last_launches += 3;
    CK(cudaEventRecord(c->ev_k[1], s));
    if (c->fwd_mma) {  // decoder MLP on the tensor cores
        const int grid_m = blocks_per_sm((const void*)shade_fwd_mma_kernel<NS, NA, true>, smem_fm) * c->sm_count;
        if (P.mode == 1)  // render: no geometry records for a backward
            shade_fwd_mma_kernel<NS, NA, false><<<grid_m, BLOCK, smem_fm, s>>>(P, W);
        else
            shade_fwd_mma_kernel<NS, NA, true><<<grid_m, BLOCK, smem_fm, s>>>(P, W);
    } else {
        const int grid_f = blocks_per_sm((const void*)shade_fwd_kernel<NS, NA, true>, smem_f) * c->sm_count;
        if (P.mode == 1)
            shade_fwd_kernel<NS, NA, false><<<grid_f, BLOCK, smem_f, s>>>(P, W);
        else
            shade_fwd_kernel<NS, NA, true><<<grid_f, BLOCK, smem_f, s>>>(P, W);
    }
    CK(cudaGetLastError());
    ++c->last_launches;
    CK(cudaEventRecord(c->ev_k[2], s));
    if (P.mode == 1) {  // render: colours of the shaded rays, no backward
        render_finish_kernel<<<4 * c->sm_count, BLOCK, 0, s>>>(P, W);
        CK(cudaGetLastError());
        ++c->last_launches;
        for (int k = 3; k <= 4; ++k) CK(cudaEventRecord(c->ev_k[k], s));
    } else {
        // the photo terms read the ground-truth colours
        run_rgb_copy(c);
        if (c->images_pending) CK(cudaStreamWaitEvent(s, c->ev_rgb, 0));
        if (c->grads_clear_pending) CK(cudaStreamWaitEvent(s, c->ev_zeroed, 0));
        const int grid_ab = blocks_per_sm((const void*)alpha_bwd_kernel, 0) * c->sm_count;
        alpha_bwd_kernel<<<grid_ab, BLOCK, 0, s>>>(P, W);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->ev_k[3], s));
        const int grid_b = blocks_per_sm((const void*)shade_bwd_kernel<NS, NA>, smem_b) * c->sm_count;
        shade_bwd_kernel<NS, NA><<<grid_b, BLOCK, smem_b, s>>>(P, W);
        CK(cudaGetLastError());
        const int grid_g = blocks_per_sm((const void*)shade_geo_kernel<NS, NA>, 0) * c->sm_count;
        shade_geo_kernel<NS, NA><<<grid_g, BLOCK, 0, s>>>(P, W);
        CK(cudaGetLastError());
        c->last_launches += 3;
        CK(cudaEventRecord(c->ev_k[4], s));
    }
    CK(cudaEventRecord(c->ev_ray1, s));
    // the pass's counters come back with the step's results
    CK(cudaMemcpyAsync(c->h_wave_counters, W.counters, sizeof(unsigned) * 8, cudaMemcpyDeviceToHost, s));
}

// Stage-0 gradient copies (psdf_set_keep_raypass_grads); (re)allocated after
// every grid upload, which frees them.
void ensure_keep_buffers(psdf_ctx* c) {
    if (!c->keep_raypass || c->d_grads0) return;
    CK(cudaMalloc(&c->d_grads0, sizeof(float) * c->n_params));
    CK(cudaMalloc(&c->d_gsmooth0, sizeof(float) * std::max<int64_t>(c->desc.T * TV, 4)));
    CK(cudaMemsetAsync(c->d_grads0, 0, sizeof(float) * c->n_params, c->stream));
    CK(cudaMemsetAsync(c->d_gsmooth0, 0, sizeof(float) * std::max<int64_t>(c->desc.T * TV, 4), c->stream));
}

// The photo terms of the rays the scan finished (stats only), on `st`.
void launch_empty_ray_loss(psdf_ctx* c, const RayPassParams& P, cudaStream_t st) {
    const int64_t n_work = P.tile_end - P.tile_begin;
    if (n_work <= 0) return;
    if (st != c->stream) CK(cudaStreamWaitEvent(st, c->ev_scanned, 0));
    run_rgb_copy(c);
    if (c->images_pending) CK(cudaStreamWaitEvent(st, c->ev_rgb, 0));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n_work + 4 * WARPS_PER_BLOCK - 1) / (4 * WARPS_PER_BLOCK),
                                                                (int64_t)8 * c->sm_count));
    empty_ray_loss_kernel<<<(unsigned)grid, BLOCK, 0, st>>>(P, c->wave, n_work);
    CK(cudaGetLastError());
    ++c->last_launches;
}

RayPassParams base_params(psdf_ctx* c) {
    RayPassParams P{};
    P.g = c->view();
    P.mlp = c->d_params + c->off_mlp;
    P.in_dim = c->in_dim;
    P.ncam = c->desc.ncam;
    P.order = c->desc.sh_order;
    P.n_max = 512;
    P.early_stop = 1e-4;
    P.bits_sm_words = c->bit_words <= kMaxSmemBitWords ? c->bit_words : 0;
    P.stage_fwd = c->stage_fwd;
    P.work_counter = c->d_work;
    P.counts = c->d_counts;
    P.stats = c->d_stats;
    return P;
}

void do_render(psdf_ctx* c, const psdf_camera* cam, const psdf_render_opts* opt, float* d_rgb,
               float* d_alpha, float* d_depth, psdf_counts* counts) {
    need_grid(c);
    if (!cam || !opt) fail(PSDF_ERR_INVALID_ARGUMENT, "null camera or options");
    check_camera(*cam);
    set_device(c);
    c->last_launches = 0;
    RayPassParams P = base_params(c);
    int order = c->desc.sh_order;  // renderer.cpp:90-91
    if (opt->sh_order_override > 0) order = std::min(opt->sh_order_override, c->desc.sh_order);
    P.order = order;
    P.no_spatial = opt->no_spatial;
    P.no_angular = opt->no_angular;
    P.no_fresnel = opt->no_fresnel;
    P.need_colors = opt->need_colors;
    P.n_max = opt->n_max;
    P.tau = opt->tau;
    P.early_stop = opt->early_stop;
    for (int i = 0; i < 3; ++i) P.bg[i] = opt->bg[i];
    std::vector<ViewDev> vd(1);
    vd[0] = ViewDev{};
    vd[0].cam = to_cam(*cam);
    vd[0].cam_bias_row = camera_bias_row(c, opt->camera_id);
    P.tile_begin = 0;
    P.tile_end = upload_viewdev(c, vd);
    P.views = c->d_viewdev;
    P.n_views = 1;
    P.out_rgb = d_rgb;
    P.out_alpha = d_alpha;
    P.out_depth = d_depth;
    // K1 through the ray-pass pipeline (scan -> composite -> decode -> finish)
    P.mode = 1;
    const int64_t n_rays = (int64_t)cam->width * cam->height;
    for (int attempt = 0;; ++attempt) {
        CK(cudaMemsetAsync(c->d_counts, 0, sizeof(unsigned long long) * 8, c->stream));
        CK(cudaMemsetAsync(c->d_stats, 0, sizeof(double) * 16, c->stream));
        prepare_sat(c, P.early_stop > 1.0 ? 0.0 : P.tau);
        dispatch_channels(c->desc.n_s, c->desc.n_a, [&]<int NS, int NA>() {
            launch_train_raypass<NS, NA>(c, P, n_rays);
        });
        if (counts) {
            CK(cudaMemcpyAsync(c->h_counts, c->d_counts, sizeof(unsigned long long) * 8,
                               cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
        if (!wave_overflowed(c)) break;
        if (attempt >= 2) fail(PSDF_ERR_RUNTIME, "ray pass buffers failed to grow");
    }
    CK(cudaEventElapsedTime(&c->last_ray_ms, c->ev_ray0, c->ev_ray1));
    c->last_step_ms = c->last_ray_ms;
    if (counts) {
        counts->n_rays = (int64_t)cam->width * cam->height;
        counts->n_marched = (int64_t)c->h_counts[1];
        counts->n_extra = (int64_t)c->h_counts[2];
        counts->n_shaded = (int64_t)c->h_counts[3];
        counts->n_alpha = 0;
        counts->n_bwd_rays = 0;
    }
}

// One train step over device-resident views (trainer.cpp:136-195).
void do_train_step(psdf_ctx* c, const std::vector<DevView*>& batch, const psdf_step_params* hp,
                   psdf_losses* losses, psdf_counts* counts, cudaEvent_t images_ready = nullptr,
                   int attempt = 0) {
    need_grid(c);
    if (!hp) fail(PSDF_ERR_INVALID_ARGUMENT, "null step parameters");
    if (batch.empty()) fail(PSDF_ERR_INVALID_ARGUMENT, "empty batch");
    set_device(c);
    c->last_launches = 0;
    cudaStream_t s = c->stream;
    CK(cudaEventRecord(c->ev_step0, s));
    // gradient clear (trainer.cpp:136).  Nothing writes a gradient before the
    // α backward / the regularizers, so with the side stream the clear runs
    // there under the saturation map and the scan (the α backward waits for
    // ev_zeroed)
    const bool overlap_clear = !c->keep_raypass;
    cudaStream_t sc = s;
    if (overlap_clear) {
        CK(cudaEventRecord(c->ev_start, s));
        CK(cudaStreamWaitEvent(c->side_stream, c->ev_start, 0));
        sc = c->side_stream;
    }
    CK(cudaMemsetAsync(c->d_grads, 0, sizeof(float) * c->n_params, sc));
    CK(cudaMemsetAsync(c->d_gsmooth, 0, sizeof(float) * c->desc.T * TV, sc));
    if (overlap_clear) CK(cudaEventRecord(c->ev_zeroed, sc));
    c->grads_clear_pending = overlap_clear;
    CK(cudaMemsetAsync(c->d_counts, 0, sizeof(unsigned long long) * 8, s));
    CK(cudaMemsetAsync(c->d_stats, 0, sizeof(double) * 16, s));

    RayPassParams P = base_params(c);
    P.tau = hp->tau;
    P.need_colors = 1;
    P.photo_scale = hp->photo_scale;
    P.bg[0] = P.bg[1] = P.bg[2] = 0.0;  // trainer uses the default background
    std::vector<ViewDev> vd(batch.size());
    int64_t n_rays = 0;
    for (size_t i = 0; i < batch.size(); ++i) {
        vd[i] = ViewDev{};
        vd[i].cam = to_cam(batch[i]->cam);
        vd[i].gt = batch[i]->rgb;
        vd[i].mask = batch[i]->mask;
        // trainer.cpp:153 + decoder.cpp:69-78
        vd[i].cam_bias_row = hp->use_camera_bias ? camera_bias_row(c, batch[i]->cam.id) : -1;
        n_rays += (int64_t)batch[i]->cam.width * batch[i]->cam.height;
    }
    // regularizers (trainer.cpp:187-191), sharded by tile / probe range.  They
    // read only parameters and the smoothed grid, so they run first (under
    // the host->device copy of the step's images when there is one) unless
    // the ray-pass-only gradients are kept for inspection.
    auto regularizers = [&](bool overlap) {
        const GridView g = c->view();
        const int T = c->desc.T, Pn = c->desc.P;
        const int t0 = (int)((int64_t)T * c->rank / c->world), t1 = (int)((int64_t)T * (c->rank + 1) / c->world);
        const int p0 = (int)((int64_t)Pn * c->rank / c->world), p1 = (int)((int64_t)Pn * (c->rank + 1) / c->world);
        const int stride = c->desc.sh_order * c->desc.sh_order * c->desc.n_a;
        // with `overlap`, the eikonal / normal / sdf kernel (the one that
        // touches only raw gradients and, atomically, the staged SDF
        // gradient) and the empty rays' photo terms run on the low-priority
        // side stream under the ray pass, filling the SMs its kernels' tails
        // leave idle (ev_fork: recorded by the ray pass after its first
        // composite round)
        cudaStream_t sl = s;
        if (overlap) {
            CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
            sl = c->side_stream;
        }
        if (t1 > t0) {
            if (c->attr_done.insert((const void*)loss_grid_kernel).second)
                CK(cudaFuncSetAttribute(loss_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kLossGridSmem));
            loss_grid_kernel<<<t1 - t0, LG_THREADS, kLossGridSmem, sl>>>(
                g, c->d_params + c->off_raw, t0, (float)hp->l_sdf, (float)hp->l_eik, (float)hp->l_norm,
                (float)(1.0 / (2.0 * c->desc.voxel_size)), c->d_gsmooth, c->d_grads + c->off_raw, c->d_stats);
            CK(cudaGetLastError());
            dispatch_ns(c->desc.n_s, [&]<int NS>() {
                loss_features_kernel<NS><<<3 * (t1 - t0), 256, 0, sl>>>(g, t0, (float)hp->l_feat,
                                                                       c->d_grads + c->off_planes, c->d_stats);
            });
            CK(cudaGetLastError());
            c->last_launches += 2;
        }
        if (p1 > p0) {
            GridMut m{g, c->d_params + c->off_raw, c->d_probe_table, c->d_probe_coords};
            const int64_t n = (int64_t)(p1 - p0) * stride;
            loss_probes_kernel<<<(unsigned)std::min<int64_t>(4 * c->sm_count, n / 256 + 1), 256, 0, sl>>>(
                m, p0, p1, stride, (float)hp->l_probe, c->d_grads + c->off_probes, c->d_stats);
            CK(cudaGetLastError());
            ++c->last_launches;
        }
        launch_empty_ray_loss(c, P, sl);
        if (overlap) CK(cudaEventRecord(c->ev_join, c->side_stream));
    };
    // the regularizers on the side stream under the ray pass, or after it on
    // the main stream (PSDF_REGS_SERIAL, A/B)
    const bool overlap = !c->keep_raypass && !c->regs_serial;
    // images still arriving (psdf_train_step): the regularizer runs under the
    // copies; resident images: under the ray pass's tail (forked by it)
    // the regularizer forks after the first composite round (it fills the
    // second round's latency tail); when it is long next to the ray pass
    // (many tiles per ray: ~1000 rays per tile or fewer, e.g. 1024^3 with a
    // 4-view batch) it forks at the step start instead (measured: 512^3
    // 3.12 vs 3.23 ms, 1024^3 5.56 vs 5.23 ms)
    const bool early = c->regs_early || (int64_t)c->desc.T * 1000 > n_rays;
    c->fork_regs = overlap && !early;
    if (overlap && early) CK(cudaEventRecord(c->ev_fork, s));
    // the saturation table needs only the grid and tau: launched before the
    // host builds the view table, so the GPU starts the step sooner
    prepare_sat(c, P.early_stop > 1.0 ? 0.0 : P.tau);
    if (images_ready) CK(cudaStreamWaitEvent(s, images_ready, 0));
    const int64_t tiles = upload_viewdev(c, vd);
    // ray-batch data parallelism: contiguous 1/N slice of the batch's work tiles
    P.tile_begin = tiles * c->rank / c->world;
    P.tile_end = tiles * (c->rank + 1) / c->world;
    P.views = c->d_viewdev;
    P.n_views = (int)vd.size();
    P.g_smooth = c->d_gsmooth;
    P.g_planes = c->d_grads + c->off_planes;
    P.g_probes = c->d_grads + c->off_probes;
    P.g_mlp = c->d_grads + c->off_mlp;
    dispatch_channels(c->desc.n_s, c->desc.n_a, [&]<int NS, int NA>() {
        launch_train_raypass<NS, NA>(c, P, n_rays);
    });
    // counts[7]: a wave buffer overflowed (summed over ranks below, so every
    // rank skips Adam and redoes the step)
    wave_overflow_kernel<<<1, 32, 0, s>>>(c->wave, c->d_counts + 7);
    CK(cudaGetLastError());
    if (c->keep_raypass) {
        ensure_keep_buffers(c);
        CK(cudaMemcpyAsync(c->d_grads0, c->d_grads, sizeof(float) * c->n_params,
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(c->d_gsmooth0, c->d_gsmooth, sizeof(float) * c->desc.T * TV,
                           cudaMemcpyDeviceToDevice, s));
    }
    c->fork_regs = false;
    regularizers(overlap);
    if (overlap) CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    // gradient exchange across ranks (GradBuffers::add, trainer.cpp:184-185,
    // across GPUs) around the G^T fold (grads.cpp:67-96: raw_grad += G^T
    // staged; Gt is linear, so each rank folds its own staged buffer):
    //  ALLREDUCE  fold, then one all-reduce of the flat gradient;
    //  BUCKETED   the [planes | probes | mlp] bucket (final once the
    //             regularizers joined) all-reduced on the comm stream under the
    //             fold, then the raw bucket;
    //  SHARDED    fold, reduce-scatter into world-size chunks, Adam on this
    //             rank's chunk only, all-gather of the updated parameters.
    const bool bucketed = c->comm && c->grad_exchange == PSDF_EXCHANGE_BUCKETED;
    const bool sharded = c->comm && c->grad_exchange == PSDF_EXCHANGE_SHARDED;
    if (bucketed) {
        CK(cudaEventRecord(c->ev_bucket, s));
        CK(cudaStreamWaitEvent(c->comm_stream, c->ev_bucket, 0));
        NK(g_nccl.AllReduce(c->d_grads + c->off_planes, c->d_grads + c->off_planes,
                            (size_t)(c->n_params - c->off_planes), ncclFloat, ncclSum, c->comm, c->comm_stream));
        CK(cudaEventRecord(c->ev_bucket_done, c->comm_stream));
    }
    launch_fold(c, c->d_gsmooth, c->d_grads + c->off_raw);
    int64_t a_lo = 0, a_n = c->n_params;  // the Adam range of this rank
    if (c->comm) {
        if (bucketed) {
            NK(g_nccl.AllReduce(c->d_grads + c->off_raw, c->d_grads + c->off_raw, (size_t)c->off_planes, ncclFloat,
                                ncclSum, c->comm, s));
            CK(cudaStreamWaitEvent(s, c->ev_bucket_done, 0));
        } else if (sharded) {
            const int64_t chunk = (c->n_params + 4 * c->world - 1) / (4 * c->world) * 4;
            a_lo = chunk * c->rank;
            a_n = std::max<int64_t>(0, std::min<int64_t>(chunk, c->n_params - a_lo));
            NK(g_nccl.ReduceScatter(c->d_grads, c->d_grads + a_lo, (size_t)chunk, ncclFloat, ncclSum, c->comm, s));
        } else {
            NK(g_nccl.AllReduce(c->d_grads, c->d_grads, (size_t)c->n_params, ncclFloat, ncclSum, c->comm, s));
        }
        NK(g_nccl.AllReduce(c->d_stats, c->d_stats, 16, ncclDouble, ncclSum, c->comm, s));
        NK(g_nccl.AllReduce(c->d_counts, c->d_counts, 8, ncclUint64, ncclSum, c->comm, s));
    }
    // Adam (trainer.cpp:194 / 53-70)
    c->adam_t += 1;
    const double c1 = 1.0 - std::pow(0.9, (double)c->adam_t);
    const double c2 = 1.0 - std::pow(0.995, (double)c->adam_t);
    if (a_n > 0) {
        adam_kernel<<<(unsigned)std::min<int64_t>(8 * c->sm_count, a_n / 1024 + 1), 256, 0, s>>>(
            c->d_params + a_lo, c->d_grads + a_lo, c->d_m + a_lo, c->d_v + a_lo, a_n, c->off_probes - a_lo,
            (float)hp->lr_vox, (float)hp->lr_mlp, (float)(1.0 / c1), (float)(1.0 / c2), c->d_counts + 7);
        CK(cudaGetLastError());
        ++c->last_launches;
    }
    if (sharded) {  // every rank's updated chunk to every rank (in place)
        const int64_t chunk = (c->n_params + 4 * c->world - 1) / (4 * c->world) * 4;
        NK(g_nccl.AllGather(c->d_params + a_lo, c->d_params, (size_t)chunk, ncclFloat, c->comm, s));
    }
    // re-smoothing (trainer.cpp:195)
    smooth_all(c);
    CK(cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(double) * 16, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_counts, c->d_counts, sizeof(unsigned long long) * 8,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(c->ev_step1, s));
    CK(cudaStreamSynchronize(s));
    if (c->h_counts[7] != 0) {  // some rank's ray pass overflowed: Adam was skipped
        c->adam_t -= 1;
        wave_overflowed(c);
        if (attempt >= 2) fail(PSDF_ERR_RUNTIME, "ray pass buffers failed to grow");
        do_train_step(c, batch, hp, losses, counts, nullptr, attempt + 1);
        return;
    }
    c->last_entries = c->h_wave_counters[0];
    c->last_records = c->h_wave_counters[5];  // sorted records (the queue minus allocation holes)
    for (int k = 0; k < 5; ++k) c->last_wave[k] = c->h_wave_counters[k];
    c->last_wave[1] = c->h_wave_counters[5];
    CK(cudaEventElapsedTime(&c->last_ray_ms, c->ev_ray0, c->ev_ray1));
    CK(cudaEventElapsedTime(&c->last_step_ms, c->ev_step0, c->ev_step1));
    for (int k = 0; k < 4; ++k) CK(cudaEventElapsedTime(&c->last_k2_ms[k], c->ev_k[k], c->ev_k[k + 1]));
    const double* st = c->h_stats;
    if (losses) {
        losses->photo = st[0];
        losses->sdf = st[3];
        losses->eik = st[4];
        losses->normal = st[5];
        losses->features = st[6];
        losses->probes = st[7];
        losses->total = st[0] + st[3] + st[4] + st[5] + st[6] + st[7];
        losses->sq_err = st[1];
        losses->mask_px = st[2];
        const double mse = st[2] > 0 ? st[1] / st[2] : 0.0;  // trainer.cpp:197-198
        losses->psnr = mse > 1e-10 ? 10.0 * std::log10(1.0 / mse) : 99.0;
    }
    if (counts) {
        counts->n_rays = n_rays;
        counts->n_marched = (int64_t)c->h_counts[1];
        counts->n_extra = (int64_t)c->h_counts[2];
        counts->n_shaded = (int64_t)c->h_counts[3];
        counts->n_alpha = (int64_t)c->h_counts[4];
        counts->n_bwd_rays = (int64_t)c->h_counts[5];
    }
}


// march_ray (renderer.cpp:55-86) for explicit rays; test hook for the
// bit-exact indexing contract.  One thread per ray.
__global__ void march_rays_kernel(GridView g, int n, const double* __restrict__ o,
                                  const double* __restrict__ d, int n_max, double* __restrict__ ts,
                                  int* __restrict__ counts) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    Marcher mr;
    int k = 0;
    if (mr.init(g, o + 3 * r, d + 3 * r, n_max)) {
        double t;
        int tile;
        while (mr.next(g, t, tile, g.tile_bits)) ts[(int64_t)r * n_max + k++] = t;
    }
    counts[r] = k;
}

// Camera::pixel_dir for every pixel (test hook).
__global__ void pixel_dirs_kernel(Cam cam, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cam.width * cam.height) return;
    const D3 d = pixel_dir(cam, (double)(i % cam.width) + 0.5, (double)(i / cam.width) + 0.5);
    out[3 * i] = d.x;
    out[3 * i + 1] = d.y;
    out[3 * i + 2] = d.z;
}

}  // namespace

// =========================================================================
extern "C" {

int psdf_abi_version(void) { return PSDF_ABI_VERSION; }

const char* psdf_last_error(psdf_ctx*) { return g_err.c_str(); }

int psdf_create(int device, psdf_ctx** out) {
    return guarded([&] {
        if (!out) fail(PSDF_ERR_INVALID_ARGUMENT, "null output pointer");
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(PSDF_ERR_INVALID_ARGUMENT, "device %d out of range (%d GPUs)", device, n);
        CK(cudaSetDevice(device));
        auto* c = new psdf_ctx;
        c->device = device;
        CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        int prio_lo = 0, prio_hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
        if (const char* e = std::getenv("PSDF_COMPOSITE_STEPS")) c->composite_steps = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("PSDF_WAVE_INIT")) c->wave_init = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("PSDF_COOP")) c->coop_round1 = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_COOP_RENDER")) c->coop_render = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_FWD_MMA")) c->fwd_mma = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_STAGE_FWD")) c->stage_fwd = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_REGS_EARLY")) c->regs_early = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_REGS_AFTER_SCAN")) c->fork_after_scan = std::atoi(e) != 0;
        if (const char* e = std::getenv("PSDF_REGS_SERIAL")) c->regs_serial = std::atoi(e) != 0;
        if (const char* m = std::getenv("PSDF_TEST_MARGIN")) c->test_margin = std::max(1e-8, std::atof(m));
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, prio_lo));
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_scanned, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_copied, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_masks, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_zeroed, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_rgb, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_rows, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_copy_free, cudaEventDisableTiming));
        CK(cudaEventRecord(c->ev_copy_free, c->stream));
        CK(cudaEventCreate(&c->ev_ray0));
        CK(cudaEventCreate(&c->ev_ray1));
        CK(cudaEventCreate(&c->ev_step0));
        CK(cudaEventCreate(&c->ev_step1));
        CK(cudaMalloc(&c->d_work, sizeof(unsigned long long) * 8));
        CK(cudaMalloc(&c->d_counts, sizeof(unsigned long long) * 8));
        CK(cudaMalloc(&c->d_stats, sizeof(double) * 16));
        CK(cudaMallocHost(&c->h_stats, sizeof(double) * 16));
        CK(cudaMallocHost(&c->h_counts, sizeof(unsigned long long) * 8));
        CK(cudaMallocHost(&c->h_wave_counters, sizeof(unsigned) * 8));
        CK(cudaMalloc(&c->wave.counters, sizeof(unsigned) * 8));
        for (auto& e : c->ev_k) CK(cudaEventCreate(&e));
        *out = c;
    });
}

int psdf_destroy(psdf_ctx* c) {
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        c->free_grid();
        for (auto& v : c->views) {
            if (v.rgb) cudaFree(v.rgb);
            if (v.mask) cudaFree(v.mask);
        }
        for (void* p : {(void*)c->d_stage_rgb, (void*)c->d_stage_mask, (void*)c->d_viewdev,
                        (void*)c->d_render, (void*)c->d_eval, (void*)c->d_mc, (void*)c->d_mesh, (void*)c->d_tmin, (void*)c->d_work, (void*)c->d_counts, (void*)c->d_stats})
            if (p) cudaFree(p);
        free_wave(c);
        if (c->wave.counters) cudaFree(c->wave.counters);
        if (c->d_tile_cnt) cudaFree(c->d_tile_cnt);
        if (c->scan_tmp) cudaFree(c->scan_tmp);
        if (c->h_wave_counters) cudaFreeHost(c->h_wave_counters);
        for (auto& e : c->ev_k) cudaEventDestroy(e);
        if (c->h_stats) cudaFreeHost(c->h_stats);
        if (c->h_counts) cudaFreeHost(c->h_counts);
        if (c->comm) g_nccl.CommDestroy(c->comm);
        if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
        if (c->ev_bucket) cudaEventDestroy(c->ev_bucket);
        if (c->ev_bucket_done) cudaEventDestroy(c->ev_bucket_done);
        cudaEventDestroy(c->ev_ray0);
        cudaEventDestroy(c->ev_ray1);
        cudaEventDestroy(c->ev_step0);
        cudaEventDestroy(c->ev_step1);
        cudaStreamDestroy(c->stream);
        cudaStreamDestroy(c->copy_stream);
        cudaStreamDestroy(c->side_stream);
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
        cudaEventDestroy(c->ev_scanned);
        cudaEventDestroy(c->ev_copied);
        cudaEventDestroy(c->ev_copy_free);
        cudaEventDestroy(c->ev_masks);
        cudaEventDestroy(c->ev_start);
        cudaEventDestroy(c->ev_zeroed);
        cudaEventDestroy(c->ev_rgb);
        cudaEventDestroy(c->ev_rows);
        if (c->d_rows) cudaFree(c->d_rows);
        if (c->h_rows) cudaFreeHost(c->h_rows);
        if (c->d_hand_bits) cudaFree(c->d_hand_bits);
        delete c;
    });
}

int64_t psdf_mlp_size(int n_s, int n_a, int ncam) {
    const int in = n_s + n_a + NPOW;
    return (int64_t)MlpLayout::make(in).cam + (int64_t)ncam * HID;
}

// Chebyshev (L-inf) distance, in tiles, from every tile to the nearest
// allocated one (0 = allocated, capped at kMaxTileDist; the marcher's
// empty-space jumps, psdf_device.cuh).  Separable: an L-inf ball is the
// product of three 1-D intervals, so three passes of
// d(x) = min_x' max(|x - x'|, d_prev(x')) over a window of kMaxTileDist.
static std::vector<uint8_t> tile_distance(const std::vector<int32_t>& tt, const int nt[3]) {
    constexpr int kMaxTileDist = 32;
    const int64_t n = (int64_t)nt[0] * nt[1] * nt[2];
    std::vector<uint8_t> a(n), b(n);
    for (int64_t i = 0; i < n; ++i) a[i] = tt[i] >= 0 ? 0 : kMaxTileDist;
    const int64_t stride[3] = {(int64_t)nt[1] * nt[2], nt[2], 1};
    for (int ax = 0; ax < 3; ++ax) {
        for (int64_t i = 0; i < n; ++i) {
            const int x = (int)((i / stride[ax]) % nt[ax]);
            int best = a[i];
            for (int r = 1; r < best; ++r) {
                if (x - r >= 0) best = std::min(best, std::max(r, (int)a[i - r * stride[ax]]));
                if (x + r < nt[ax]) best = std::min(best, std::max(r, (int)a[i + r * stride[ax]]));
            }
            b[i] = (uint8_t)best;
        }
        a.swap(b);
    }
    return a;
}

// Fresh-tile defaults generated on the device instead of uploaded: planes =
// value in the first hs channels (zero in padded ones), probes = 0.
struct FreshFill {
    float plane_value;
    int plane_hs;
};

// The device upload proper: d is in device layout (kernel widths); raw, smooth,
// planes and probes may be device pointers (copies are cudaMemcpyDefault).
static void upload_grid_dev(psdf_ctx* c, const psdf_grid_desc* d, const int32_t* tile_coords,
                            const int32_t* probe_ids, const int32_t* probe_coords, const float* raw,
                            const float* smooth, const float* planes, const float* probes,
                            const FreshFill* fresh = nullptr) {
    {
        if (!c || !d) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        for (int a = 0; a < 3; ++a)
            if (d->res[a] <= 0 || d->res[a] % TE)
                fail(PSDF_ERR_INVALID_ARGUMENT, "grid resolution must be a multiple of 16");
        if (d->sh_order < 1 || d->sh_order > 4)
            fail(PSDF_ERR_INVALID_ARGUMENT, "SH order must be in [1,4]");
        if (!supported_channels(d->n_s, d->n_a))
            fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported kernel widths (n_s, n_a) = (%d, %d)", d->n_s, d->n_a);
        if (d->T < 0 || d->P < 0 || d->ncam < 0) fail(PSDF_ERR_INVALID_ARGUMENT, "negative count");
        if (d->T > 0 && (!tile_coords || !probe_ids || !raw || (!planes && !fresh)))
            fail(PSDF_ERR_INVALID_ARGUMENT, "missing tile arrays");
        if (d->P > 0 && (!probe_coords || (!probes && !fresh)))
            fail(PSDF_ERR_INVALID_ARGUMENT, "missing probe arrays");
        set_device(c);
        CK(cudaStreamSynchronize(c->stream));
        c->free_grid();
        c->desc = *d;
        c->in_dim = d->n_s + d->n_a + NPOW;
        for (int a = 0; a < 3; ++a) {
            c->occ_tlo[a] = 0;
            c->occ_thi[a] = -1;
        }
        for (int a = 0; a < 3; ++a) c->nt[a] = d->res[a] / TE;
        const int64_t T = d->T, P = d->P;
        // dense tile / probe lattice tables
        const int64_t ntt = (int64_t)c->nt[0] * c->nt[1] * c->nt[2];
        const int64_t npt = (int64_t)(c->nt[0] + 1) * (c->nt[1] + 1) * (c->nt[2] + 1);
        std::vector<int32_t> tt(ntt, -1), pt(npt, -1);
        std::vector<int4> tc4(std::max<int64_t>(T, 1)), pc4(std::max<int64_t>(P, 1));
        for (int64_t t = 0; t < T; ++t) {
            const int32_t* q = tile_coords + 3 * t;
            for (int a = 0; a < 3; ++a)
                if (q[a] < 0 || q[a] >= c->nt[a]) fail(PSDF_ERR_INVALID_ARGUMENT, "tile %lld outside the grid", (long long)t);
            int32_t& slot = tt[((int64_t)q[0] * c->nt[1] + q[1]) * c->nt[2] + q[2]];
            if (slot >= 0) fail(PSDF_ERR_INVALID_ARGUMENT, "duplicate tile coordinates");
            slot = (int32_t)t;
            tc4[t] = make_int4(q[0], q[1], q[2], 0);
            for (int a = 0; a < 3; ++a) {
                if (t == 0 || q[a] < c->occ_tlo[a]) c->occ_tlo[a] = q[a];
                if (t == 0 || q[a] > c->occ_thi[a]) c->occ_thi[a] = q[a];
            }
            for (int i = 0; i < 8; ++i)
                if (probe_ids[8 * t + i] < 0 || probe_ids[8 * t + i] >= P)
                    fail(PSDF_ERR_INVALID_ARGUMENT, "probe id out of range");
        }
        for (int64_t p = 0; p < P; ++p) {
            const int32_t* q = probe_coords + 3 * p;
            for (int a = 0; a < 3; ++a)
                if (q[a] < 0 || q[a] > c->nt[a]) fail(PSDF_ERR_INVALID_ARGUMENT, "probe %lld outside the lattice", (long long)p);
            pt[((int64_t)q[0] * (c->nt[1] + 1) + q[1]) * (c->nt[2] + 1) + q[2]] = (int32_t)p;
            pc4[p] = make_int4(q[0], q[1], q[2], 0);
        }
        const int nc = d->sh_order * d->sh_order;
        c->n_planes = T * 3 * 256 * d->n_s;
        c->n_probes = P * nc * d->n_a;
        c->mlp_size = psdf_mlp_size(d->n_s, d->n_a, d->ncam);
        c->off_raw = 0;
        c->off_planes = up4(T * TV);
        c->off_probes = up4(c->off_planes + c->n_planes);
        c->off_mlp = up4(c->off_probes + c->n_probes);
        c->n_params = up4(c->off_mlp + c->mlp_size);
        CK(cudaMalloc(&c->d_tile_table, sizeof(int32_t) * ntt));
        c->bit_words = (int)((ntt + 31) / 32);
        std::vector<uint32_t> bits(c->bit_words, 0u);
        for (int64_t i = 0; i < ntt; ++i)
            if (tt[i] >= 0) bits[i >> 5] |= 1u << (i & 31);
        CK(cudaMalloc(&c->d_tile_bits, sizeof(uint32_t) * c->bit_words));
        CK(cudaMemcpyAsync(c->d_tile_bits, bits.data(), sizeof(uint32_t) * c->bit_words,
                           cudaMemcpyHostToDevice, c->stream));
        const std::vector<uint8_t> dist = tile_distance(tt, c->nt);
        std::vector<int32_t> nbr(27 * std::max<int64_t>(T, 1), -1);
        for (int64_t t = 0; t < T; ++t)
            for (int k = 0; k < 27; ++k) {
                const int q[3] = {tc4[t].x + k / 9 - 1, tc4[t].y + (k / 3) % 3 - 1, tc4[t].z + k % 3 - 1};
                if (q[0] >= 0 && q[1] >= 0 && q[2] >= 0 && q[0] < c->nt[0] && q[1] < c->nt[1] && q[2] < c->nt[2])
                    nbr[27 * t + k] = tt[((int64_t)q[0] * c->nt[1] + q[1]) * c->nt[2] + q[2]];
            }
        CK(cudaMalloc(&c->d_tile_nbr, sizeof(int32_t) * nbr.size()));
        CK(cudaMemcpyAsync(c->d_tile_nbr, nbr.data(), sizeof(int32_t) * nbr.size(), cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaMalloc(&c->d_tile_dist, std::max<int64_t>(ntt, 1)));
        CK(cudaMemcpyAsync(c->d_tile_dist, dist.data(), ntt, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // the host vectors above are about to go
        CK(cudaMalloc(&c->d_probe_table, sizeof(int32_t) * npt));
        CK(cudaMalloc(&c->d_tile_coords, sizeof(int4) * tc4.size()));
        CK(cudaMalloc(&c->d_probe_coords, sizeof(int4) * pc4.size()));
        CK(cudaMalloc(&c->d_probe_ids, sizeof(int32_t) * std::max<int64_t>(8 * T, 1)));
        CK(cudaMalloc(&c->d_params, sizeof(float) * (c->n_params + kParamPad)));
        CK(cudaMalloc(&c->d_grads, sizeof(float) * (c->n_params + kParamPad)));
        CK(cudaMalloc(&c->d_m, sizeof(float) * (c->n_params + kParamPad)));
        CK(cudaMalloc(&c->d_v, sizeof(float) * (c->n_params + kParamPad)));
        CK(cudaMalloc(&c->d_smooth, sizeof(float) * std::max<int64_t>(T * TV, 4)));
        CK(cudaMalloc(&c->d_smooth_ap, sizeof(float) * std::max<int64_t>(T * AV, 4)));
        CK(cudaMalloc(&c->d_sat_dist, std::max<int64_t>((int64_t)kCellN * T, 1)));
        c->sat_ok = false;
        CK(cudaMalloc(&c->d_gsmooth, sizeof(float) * std::max<int64_t>(T * TV, 4)));
        CK(cudaMemsetAsync(c->d_params, 0, sizeof(float) * (c->n_params + kParamPad), c->stream));
        CK(cudaMemsetAsync(c->d_grads, 0, sizeof(float) * (c->n_params + kParamPad), c->stream));
        CK(cudaMemsetAsync(c->d_m, 0, sizeof(float) * (c->n_params + kParamPad), c->stream));
        CK(cudaMemsetAsync(c->d_v, 0, sizeof(float) * (c->n_params + kParamPad), c->stream));
        CK(cudaMemcpyAsync(c->d_tile_table, tt.data(), sizeof(int32_t) * ntt, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->d_probe_table, pt.data(), sizeof(int32_t) * npt, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->d_tile_coords, tc4.data(), sizeof(int4) * tc4.size(), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->d_probe_coords, pc4.data(), sizeof(int4) * pc4.size(), cudaMemcpyHostToDevice, c->stream));
        if (T > 0) {
            CK(cudaMemcpyAsync(c->d_probe_ids, probe_ids, sizeof(int32_t) * 8 * T, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(c->d_params + c->off_raw, raw, sizeof(float) * T * TV, cudaMemcpyDefault, c->stream));
            if (planes) {
                CK(cudaMemcpyAsync(c->d_params + c->off_planes, planes, sizeof(float) * c->n_planes,
                                   cudaMemcpyDefault, c->stream));
            } else {
                const unsigned nb = (unsigned)std::min<int64_t>((c->n_planes + 255) / 256, 8 * c->sm_count);
                plane_fill_kernel<<<nb, 256, 0, c->stream>>>(c->d_params + c->off_planes, c->n_planes, d->n_s,
                                                             fresh->plane_hs, fresh->plane_value);
                CK(cudaGetLastError());
            }
        }
        if (P > 0 && probes)  // fresh probes: the zeroed buffer
            CK(cudaMemcpyAsync(c->d_params + c->off_probes, probes, sizeof(float) * c->n_probes,
                               cudaMemcpyDefault, c->stream));
        c->has_grid = true;
        c->adam_t = 0;
        if (smooth && T > 0) {
            CK(cudaMemcpyAsync(c->d_smooth, smooth, sizeof(float) * T * TV, cudaMemcpyDefault, c->stream));
            fill_apron(c);
        } else {
            smooth_all(c);
        }
        CK(cudaStreamSynchronize(c->stream));
    }
}

// SparseGrid upload in the caller's layout (psdf.h); widths without their own
// kernel instantiation are zero-padded to kernel_widths().
int psdf_upload_grid(psdf_ctx* c, const psdf_grid_desc* d, const int32_t* tile_coords,
                     const int32_t* probe_ids, const int32_t* probe_coords, const float* raw,
                     const float* smooth, const float* planes, const float* probes) {
    return guarded([&] {
        if (!c || !d) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        int ks = 0, ka = 0;
        if (!kernel_widths(d->n_s, d->n_a, &ks, &ka))
            fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported (n_s, n_a) = (%d, %d)", d->n_s, d->n_a);
        if (ks == d->n_s && ka == d->n_a) {
            upload_grid_dev(c, d, tile_coords, probe_ids, probe_coords, raw, smooth, planes, probes);
        } else {
            if (d->T < 0 || d->P < 0 || d->sh_order < 1 || d->sh_order > 4)
                fail(PSDF_ERR_INVALID_ARGUMENT, "invalid grid counts or SH order");
            psdf_grid_desc dk = *d;
            dk.n_s = ks;
            dk.n_a = ka;
            const int64_t nc = (int64_t)d->sh_order * d->sh_order;
            std::vector<float> pl, pr;
            if (planes) {
                pl.resize((size_t)d->T * 3 * 256 * ks);
                repack_rows(planes, (int64_t)d->T * 3 * 256, d->n_s, pl.data(), ks);
            }
            if (probes) {
                pr.resize((size_t)d->P * nc * ka);
                repack_rows(probes, (int64_t)d->P * nc, d->n_a, pr.data(), ka);
            }
            upload_grid_dev(c, &dk, tile_coords, probe_ids, probe_coords, raw, smooth,
                            planes ? pl.data() : nullptr, probes ? pr.data() : nullptr);
        }
        c->hns = d->n_s;
        c->hna = d->n_a;
    });
}

// MLP blob in device layout (kernel widths)
static void upload_mlp_dev(psdf_ctx* c, const float* mlp, int64_t n) {
    need_grid(c);
    if (!mlp || n != c->mlp_size)
        fail(PSDF_ERR_INVALID_ARGUMENT, "MLP size %lld does not match the grid (%lld)",
             (long long)n, (long long)c->mlp_size);
    set_device(c);
    CK(cudaMemcpyAsync(c->d_params + c->off_mlp, mlp, sizeof(float) * n, cudaMemcpyDefault, c->stream));
    CK(cudaStreamSynchronize(c->stream));
}

static bool padded(const psdf_ctx* c) { return c->hns != c->desc.n_s || c->hna != c->desc.n_a; }

int psdf_upload_mlp(psdf_ctx* c, const float* mlp, int64_t n) {
    return guarded([&] {
        need_grid(c);
        if (!padded(c)) return upload_mlp_dev(c, mlp, n);
        const int64_t nh = psdf_mlp_size(c->hns, c->hna, c->desc.ncam);
        if (!mlp || n != nh)
            fail(PSDF_ERR_INVALID_ARGUMENT, "MLP size %lld does not match the grid (%lld)", (long long)n,
                 (long long)nh);
        std::vector<float> k((size_t)c->mlp_size);
        repack_mlp(mlp, c->hns, c->hna, k.data(), c->desc.n_s, c->desc.n_a, c->desc.ncam);
        upload_mlp_dev(c, k.data(), (int64_t)k.size());
    });
}

// Parameters (or gradients: base / smooth_src) in device layout.
static void download_params_dev(psdf_ctx* c, const float* base, const float* smooth_src, float* raw, float* smooth,
                                float* planes, float* probes, float* mlp) {
    need_grid(c);
    set_device(c);
    const int64_t T = c->desc.T;
    cudaStream_t s = c->stream;
    if (raw && T) CK(cudaMemcpyAsync(raw, base + c->off_raw, sizeof(float) * T * TV, cudaMemcpyDeviceToHost, s));
    if (smooth && T) CK(cudaMemcpyAsync(smooth, smooth_src, sizeof(float) * T * TV, cudaMemcpyDeviceToHost, s));
    if (planes && T) CK(cudaMemcpyAsync(planes, base + c->off_planes, sizeof(float) * c->n_planes, cudaMemcpyDeviceToHost, s));
    if (probes && c->n_probes) CK(cudaMemcpyAsync(probes, base + c->off_probes, sizeof(float) * c->n_probes, cudaMemcpyDeviceToHost, s));
    if (mlp) CK(cudaMemcpyAsync(mlp, base + c->off_mlp, sizeof(float) * c->mlp_size, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

// The same in the caller's layout: padded channels stripped.
static void download_params_host(psdf_ctx* c, const float* base, const float* smooth_src, float* raw,
                                 float* smooth, float* planes, float* probes, float* mlp) {
    need_grid(c);
    if (!padded(c)) return download_params_dev(c, base, smooth_src, raw, smooth, planes, probes, mlp);
    std::vector<float> pl(planes ? c->n_planes : 0), pr(probes ? c->n_probes : 0), ml(mlp ? c->mlp_size : 0);
    download_params_dev(c, base, smooth_src, raw, smooth, planes ? pl.data() : nullptr,
                        probes ? pr.data() : nullptr, mlp ? ml.data() : nullptr);
    const psdf_grid_desc& d = c->desc;
    if (planes) repack_rows(pl.data(), (int64_t)d.T * 3 * 256, d.n_s, planes, c->hns);
    if (probes) repack_rows(pr.data(), (int64_t)d.P * d.sh_order * d.sh_order, d.n_a, probes, c->hna);
    if (mlp) repack_mlp(ml.data(), d.n_s, d.n_a, mlp, c->hns, c->hna, d.ncam);
}

int psdf_download_params(psdf_ctx* c, float* raw, float* smooth, float* planes, float* probes,
                         float* mlp) {
    return guarded([&] {
        need_grid(c);
        download_params_host(c, c->d_params, c->d_smooth, raw, smooth, planes, probes, mlp);
    });
}

int psdf_grid_info(psdf_ctx* c, psdf_grid_desc* out) {
    return guarded([&] {
        need_grid(c);
        if (!out) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        *out = c->desc;
        out->n_s = c->hns;  // the caller's widths
        out->n_a = c->hna;
    });
}

int psdf_download_structure(psdf_ctx* c, int32_t* tile_coords, int32_t* probe_ids, int32_t* probe_coords) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        const int64_t T = c->desc.T, P = c->desc.P;
        std::vector<int4> tc(std::max<int64_t>(T, 1)), pc(std::max<int64_t>(P, 1));
        if (T) CK(cudaMemcpy(tc.data(), c->d_tile_coords, sizeof(int4) * T, cudaMemcpyDeviceToHost));
        if (P) CK(cudaMemcpy(pc.data(), c->d_probe_coords, sizeof(int4) * P, cudaMemcpyDeviceToHost));
        if (probe_ids && T) CK(cudaMemcpy(probe_ids, c->d_probe_ids, sizeof(int32_t) * 8 * T, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; tile_coords && t < T; ++t) {
            tile_coords[3 * t] = tc[t].x;
            tile_coords[3 * t + 1] = tc[t].y;
            tile_coords[3 * t + 2] = tc[t].z;
        }
        for (int64_t p = 0; probe_coords && p < P; ++p) {
            probe_coords[3 * p] = pc[p].x;
            probe_coords[3 * p + 1] = pc[p].y;
            probe_coords[3 * p + 2] = pc[p].z;
        }
    });
}

// SparseGrid::raise_sh_order (grid.cpp:252-262): band-major probes, the new
// bands start at zero.  Re-lays the parameter buffer out (the optimizer state
// is reset, as the reference rebuilds it every LOD, trainer.cpp:115).
int psdf_raise_sh_order(psdf_ctx* c, int new_order) {
    return guarded([&] {
        need_grid(c);
        if (new_order < c->desc.sh_order || new_order > 4)
            fail(PSDF_ERR_INVALID_ARGUMENT, "raise_sh_order: order must not decrease and must be <= 4");
        if (new_order == c->desc.sh_order) return;
        set_device(c);
        cudaStream_t s = c->stream;
        psdf_grid_desc d = c->desc;
        const int64_t T = d.T, P = d.P;
        std::vector<int32_t> tc(3 * std::max<int64_t>(T, 1)), pid(8 * std::max<int64_t>(T, 1)),
            pco(3 * std::max<int64_t>(P, 1));
        if (psdf_download_structure(c, tc.data(), pid.data(), pco.data()) != PSDF_OK)
            fail(PSDF_ERR_RUNTIME, "%s", g_err.c_str());
        // raw / smoothed SDF, planes and MLP are unchanged: device copies;
        // the (small) probe pool is re-laid out band-major on the host
        DevScratch scratch;
        float* d_raw = scratch.alloc<float>((size_t)T * TV);
        float* d_sm = scratch.alloc<float>((size_t)T * TV);
        float* d_planes = scratch.alloc<float>((size_t)c->n_planes);
        float* d_mlp = scratch.alloc<float>((size_t)c->mlp_size);
        const int64_t n_mlp = c->mlp_size;
        if (T) {
            CK(cudaMemcpyAsync(d_raw, c->d_params + c->off_raw, sizeof(float) * T * TV, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(d_sm, c->d_smooth, sizeof(float) * T * TV, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(d_planes, c->d_params + c->off_planes, sizeof(float) * c->n_planes,
                               cudaMemcpyDeviceToDevice, s));
        }
        CK(cudaMemcpyAsync(d_mlp, c->d_params + c->off_mlp, sizeof(float) * n_mlp, cudaMemcpyDeviceToDevice, s));
        std::vector<float> probes(c->n_probes);
        if (c->n_probes)
            CK(cudaMemcpyAsync(probes.data(), c->d_params + c->off_probes, sizeof(float) * c->n_probes,
                               cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int oc = d.sh_order * d.sh_order * d.n_a, nc = new_order * new_order * d.n_a;
        std::vector<float> np((size_t)P * nc, 0.f);
        for (int64_t p = 0; p < P; ++p)
            std::copy(probes.begin() + p * oc, probes.begin() + (p + 1) * oc, np.begin() + p * nc);
        d.sh_order = new_order;
        upload_grid_dev(c, &d, tc.data(), pid.data(), pco.data(), d_raw, T ? d_sm : nullptr, d_planes, np.data());
        upload_mlp_dev(c, d_mlp, n_mlp);
    });
}

// SparseGrid::subdivide (grid.cpp:271-345) on the device: child raw values,
// allocation decisions, plane upsampling and probe re-interpolation are
// kernels (psdf_lod.cuh); the new tile / probe lists are built on the host in
// the reference's allocate_tile / ensure_probe order, and the new grid is
// then uploaded (smoothed on the device, optimizer state reset).
int psdf_subdivide(psdf_ctx* c, double band_voxels, int32_t* out_T, int32_t* out_P) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        cudaStream_t s = c->stream;
        const psdf_grid_desc d0 = c->desc;
        const int64_t T0 = d0.T;
        psdf_grid_desc d = d0;
        d.voxel_size = d0.voxel_size * 0.5;
        for (int a = 0; a < 3; ++a) d.res[a] = d0.res[a] * 2;
        const int nt1[3] = {d.res[0] / TE, d.res[1] / TE, d.res[2] / TE};
        // 1. child raw values + allocation decisions
        DevScratch scratch;
        float* d_child = scratch.alloc<float>((size_t)TV * 8 * T0);
        uint8_t* d_keep = scratch.alloc<uint8_t>((size_t)8 * T0);
        std::vector<uint8_t> keep(8 * T0);
        std::vector<int4> tc0(std::max<int64_t>(T0, 1));
        if (T0) {
            subdiv_raw_kernel<<<(unsigned)(8 * T0), 256, 0, s>>>(c->view(), c->d_params + c->off_raw, d.voxel_size,
                                                               band_voxels * d.voxel_size, d_child, d_keep);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(keep.data(), d_keep, 8 * T0, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(tc0.data(), c->d_tile_coords, sizeof(int4) * T0, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        // 2. new tiles in the reference's order (parent order, child 0..7),
        //    probes by first touch (allocate_tile -> ensure_probe)
        std::vector<int32_t> tc, pid, pco;
        std::vector<int> src;
        std::unordered_map<int64_t, int> probe_of;
        auto key = [&](int x, int y, int z) { return ((int64_t)x * (nt1[1] + 1) + y) * (nt1[2] + 1) + z; };
        for (int64_t t = 0; t < T0; ++t)
            for (int ch = 0; ch < 8; ++ch) {
                if (!keep[8 * t + ch]) continue;
                const int q[3] = {2 * tc0[t].x + (ch & 1), 2 * tc0[t].y + ((ch >> 1) & 1), 2 * tc0[t].z + ((ch >> 2) & 1)};
                tc.insert(tc.end(), q, q + 3);
                src.push_back((int)(8 * t + ch));
                for (int i = 0; i < 8; ++i) {
                    const int g[3] = {q[0] + (i & 1), q[1] + ((i >> 1) & 1), q[2] + ((i >> 2) & 1)};
                    auto it = probe_of.find(key(g[0], g[1], g[2]));
                    int id;
                    if (it == probe_of.end()) {
                        id = (int)(pco.size() / 3);
                        probe_of.emplace(key(g[0], g[1], g[2]), id);
                        pco.insert(pco.end(), g, g + 3);
                    } else {
                        id = it->second;
                    }
                    pid.push_back(id);
                }
            }
        const int64_t T1 = (int64_t)src.size(), P1 = (int64_t)(pco.size() / 3);
        d.T = (int)T1;
        d.P = (int)P1;
        // 3. resampled parameters on the device
        const int stride = d0.sh_order * d0.sh_order * d0.n_a;
        std::vector<int4> pc4(std::max<int64_t>(P1, 1));
        for (int64_t p = 0; p < P1; ++p) pc4[p] = make_int4(pco[3 * p], pco[3 * p + 1], pco[3 * p + 2], 0);
        int* d_src = scratch.alloc<int>((size_t)T1);
        int4* d_pc = scratch.alloc<int4>((size_t)P1);
        float* d_raw = scratch.alloc<float>((size_t)TV * T1);
        float* d_planes = scratch.alloc<float>((size_t)3 * 256 * d0.n_s * T1);
        float* d_probes = scratch.alloc<float>((size_t)stride * P1);
        if (T1) CK(cudaMemcpyAsync(d_src, src.data(), sizeof(int) * T1, cudaMemcpyHostToDevice, s));
        if (P1) CK(cudaMemcpyAsync(d_pc, pc4.data(), sizeof(int4) * P1, cudaMemcpyHostToDevice, s));
        if (T1) {
            subdiv_gather_raw_kernel<<<(unsigned)T1, 256, 0, s>>>(d_child, d_src, (int)T1, d_raw);
            CK(cudaGetLastError());
            subdiv_planes_kernel<<<(unsigned)T1, 256, 0, s>>>(c->d_params + c->off_planes, d0.n_s, d_src, (int)T1,
                                                             d_planes);
            CK(cudaGetLastError());
        }
        if (P1) {
            const int3 pdim = make_int3(c->nt[0] + 1, c->nt[1] + 1, c->nt[2] + 1);
            subdiv_probes_kernel<<<(unsigned)P1, 128, 0, s>>>(c->d_probe_table, pdim, c->d_params + c->off_probes,
                                                              stride, d_pc, (int)P1, d_probes);
            CK(cudaGetLastError());
        }
        const int64_t n_mlp = c->mlp_size;
        float* d_mlp = scratch.alloc<float>((size_t)n_mlp);
        CK(cudaMemcpyAsync(d_mlp, c->d_params + c->off_mlp, sizeof(float) * n_mlp, cudaMemcpyDeviceToDevice, s));
        // 4. the new grid (smoothed on the device, grid.cpp:340), uploaded
        // device to device from the resampled buffers
        upload_grid_dev(c, &d, tc.data(), pid.data(), pco.data(), d_raw, nullptr, d_planes, d_probes);
        upload_mlp_dev(c, d_mlp, n_mlp);
        scratch.release();
        if (out_T) *out_T = (int32_t)T1;
        if (out_P) *out_P = (int32_t)P1;
    });
}

// init_grid_visual_hull (grid.cpp:470-504) on the device: occupancy,
// two squared EDTs, the seed SDF and the per-tile allocation decision are
// kernels (psdf_lod.cuh); the tile / probe lists are built on the host in
// init_common's order (tiles x-major, allocate_tile -> ensure_probe), then
// uploaded with the reference's defaults (planes 0.5, probes 0, smoothed on
// the device).  The MLP is zero until psdf_upload_mlp.
int psdf_init_visual_hull(psdf_ctx* c, const psdf_grid_desc* cfg, int band_voxels, int n_cams,
                          const psdf_camera* cams, const uint8_t* const* masks, int32_t* out_T, int32_t* out_P) {
    return guarded([&] {
        if (!c || !cfg) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        if (n_cams <= 0 || !cams || !masks) fail(PSDF_ERR_INVALID_ARGUMENT, "visual hull: need one mask per camera");
        int ks0 = 0, ka0 = 0;
        if (!kernel_widths(cfg->n_s, cfg->n_a, &ks0, &ka0))
            fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported (n_s, n_a) = (%d, %d)", cfg->n_s, cfg->n_a);
        for (int a = 0; a < 3; ++a)
            if (cfg->res[a] <= 0 || cfg->res[a] % TE)
                fail(PSDF_ERR_INVALID_ARGUMENT, "grid resolution must be a multiple of 16");
        for (int i = 0; i < n_cams; ++i) {
            check_camera(cams[i]);
            if (!masks[i]) fail(PSDF_ERR_INVALID_ARGUMENT, "visual hull: need one mask per camera");
        }
        set_device(c);
        cudaStream_t s = c->stream;
        const int3 res = make_int3(cfg->res[0], cfg->res[1], cfg->res[2]);
        const int64_t nv = (int64_t)res.x * res.y * res.z;
        const double h = cfg->voxel_size;
        // one call-scoped arena for every temporary (sizes known up front)
        const int maxn = std::max({res.x, res.y, res.z});
        const int64_t n_lines_max = std::max({(int64_t)res.x * res.y, (int64_t)res.x * res.z, (int64_t)res.y * res.z});
        const int batch = (int)std::min<int64_t>(n_lines_max, 131072);
        const int nt[3] = {res.x / TE, res.y / TE, res.z / TE};
        const int64_t ntt = (int64_t)nt[0] * nt[1] * nt[2];
        size_t mask_bytes = 0;
        for (int i = 0; i < n_cams; ++i) mask_bytes += ((size_t)cams[i].width * cams[i].height + 255) & ~(size_t)255;
        auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
        const size_t arena_bytes = mask_bytes + al(sizeof(Cam) * n_cams) + al(sizeof(uint8_t*) * n_cams) + al(nv) +
                                   al(sizeof(double) * (size_t)batch * maxn) + al(sizeof(int) * (size_t)batch * maxn) +
                                   al(sizeof(double) * (size_t)batch * (maxn + 1)) + 2 * al(sizeof(double) * nv) +
                                   al(sizeof(float) * TV * ntt) + al(ntt) + al(sizeof(int) * ntt);
        DevScratch scratch;
        uint8_t* arena = scratch.alloc<uint8_t>(arena_bytes);
        size_t used = 0;
        auto dalloc = [&](size_t bytes) {
            void* p = arena + used;
            used += al(bytes);
            if (used > arena_bytes) fail(PSDF_ERR_RUNTIME, "visual hull: scratch arena overflow");
            return p;
        };
        {
            // cameras and masks
            std::vector<Cam> hc(n_cams);
            std::vector<const uint8_t*> hm(n_cams);
            for (int i = 0; i < n_cams; ++i) {
                hc[i] = to_cam(cams[i]);
                const size_t n = (size_t)cams[i].width * cams[i].height;
                auto* dm = (uint8_t*)dalloc(n);
                CK(cudaMemcpyAsync(dm, masks[i], n, cudaMemcpyHostToDevice, s));
                hm[i] = dm;
            }
            auto* d_cams = (Cam*)dalloc(sizeof(Cam) * n_cams);
            auto* d_masks = (const uint8_t**)dalloc(sizeof(uint8_t*) * n_cams);
            CK(cudaMemcpyAsync(d_cams, hc.data(), sizeof(Cam) * n_cams, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_masks, hm.data(), sizeof(uint8_t*) * n_cams, cudaMemcpyHostToDevice, s));
            // occupancy (grid.cpp:477-491)
            auto* occ = (uint8_t*)dalloc(nv);
            const unsigned gv = (unsigned)std::min<int64_t>((nv + 255) / 256, 64 * c->sm_count);
            hull_occ_kernel<<<gv, 256, 0, s>>>(d_cams, d_masks, n_cams, res,
                                               make_double3(cfg->origin[0], cfg->origin[1], cfg->origin[2]), h, occ);
            CK(cudaGetLastError());
            // squared EDTs to the occupied and to the free set (edt3d, grid.cpp:430-468)
            auto* fbuf = (double*)dalloc(sizeof(double) * (size_t)batch * maxn);
            auto* vbuf = (int*)dalloc(sizeof(int) * (size_t)batch * maxn);
            auto* zbuf = (double*)dalloc(sizeof(double) * (size_t)batch * (maxn + 1));
            const int64_t syz = (int64_t)res.y * res.z;
            const EdtLines passes[3] = {
                {res.x * res.y, res.z, 1, syz, res.z, res.y},          // along z, lines (x, y)
                {res.x * res.z, res.y, res.z, syz, 1, res.z},          // along y, lines (x, z)
                {res.y * res.z, res.x, (int)syz, res.z, 1, res.z}};    // along x, lines (y, z)
            double* dist[2];
            for (int w = 0; w < 2; ++w) {
                dist[w] = (double*)dalloc(sizeof(double) * nv);
                edt_init_kernel<<<gv, 256, 0, s>>>(occ, nv, w == 0 ? 1 : 0, dist[w]);
                CK(cudaGetLastError());
                for (const EdtLines& L : passes)
                    for (int l0 = 0; l0 < L.n_lines; l0 += batch) {
                        edt_pass_kernel<<<(batch + 127) / 128, 128, 0, s>>>(dist[w], L, l0, batch, fbuf, vbuf, zbuf);
                        CK(cudaGetLastError());
                    }
            }
            // seed SDF + allocation decision per tile (init_common, grid.cpp:358-397)
            auto* raw_all = (float*)dalloc(sizeof(float) * TV * ntt);
            auto* keep_d = (uint8_t*)dalloc(ntt);
            const double max_s = (double)maxn * h;
            hull_tiles_kernel<<<(unsigned)ntt, 256, 0, s>>>(dist[0], dist[1], res, h, max_s, band_voxels * h, raw_all,
                                                            keep_d);
            CK(cudaGetLastError());
            std::vector<uint8_t> keep(ntt);
            CK(cudaMemcpyAsync(keep.data(), keep_d, ntt, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<int32_t> tc, pid, pco;
            std::vector<int> src;
            std::unordered_map<int64_t, int> probe_of;
            auto key = [&](int x, int y, int z) { return ((int64_t)x * (nt[1] + 1) + y) * (nt[2] + 1) + z; };
            for (int64_t t = 0; t < ntt; ++t) {
                if (!keep[t]) continue;
                const int q[3] = {(int)(t / ((int64_t)nt[1] * nt[2])), (int)((t / nt[2]) % nt[1]), (int)(t % nt[2])};
                tc.insert(tc.end(), q, q + 3);
                src.push_back((int)t);
                for (int i = 0; i < 8; ++i) {
                    const int g[3] = {q[0] + (i & 1), q[1] + ((i >> 1) & 1), q[2] + ((i >> 2) & 1)};
                    auto it = probe_of.find(key(g[0], g[1], g[2]));
                    int id;
                    if (it == probe_of.end()) {
                        id = (int)(pco.size() / 3);
                        probe_of.emplace(key(g[0], g[1], g[2]), id);
                        pco.insert(pco.end(), g, g + 3);
                    } else {
                        id = it->second;
                    }
                    pid.push_back(id);
                }
            }
            const int64_t T = (int64_t)src.size(), P = (int64_t)(pco.size() / 3);
            // the kept tiles' raw values, gathered on the device into the
            // (finished) occupied-set EDT buffer and uploaded from there
            float* d_raw = reinterpret_cast<float*>(dist[0]);
            if (T) {
                auto* d_src = (int*)dalloc(sizeof(int) * T);
                CK(cudaMemcpyAsync(d_src, src.data(), sizeof(int) * T, cudaMemcpyHostToDevice, s));
                subdiv_gather_raw_kernel<<<(unsigned)T, 256, 0, s>>>(raw_all, d_src, (int)T, d_raw);
                CK(cudaGetLastError());
            }
            psdf_grid_desc d = *cfg;
            d.T = (int)T;
            d.P = (int)P;
            int ks = 0, ka = 0;
            if (!kernel_widths(d.n_s, d.n_a, &ks, &ka))
                fail(PSDF_ERR_INVALID_ARGUMENT, "unsupported (n_s, n_a) = (%d, %d)", d.n_s, d.n_a);
            psdf_grid_desc dk = d;
            dk.n_s = ks;
            dk.n_a = ka;
            // planes 0.5 (allocate_tile, grid.cpp:66-69), probes 0
            // (ensure_probe), MLP 0 until psdf_upload_mlp: generated on the
            // device; the raw copy is device to device
            const FreshFill fresh{0.5f, d.n_s};
            upload_grid_dev(c, &dk, tc.data(), pid.data(), pco.data(), d_raw, nullptr, nullptr, nullptr, &fresh);
            c->hns = d.n_s;
            c->hna = d.n_a;
            if (out_T) *out_T = (int32_t)T;
            if (out_P) *out_P = (int32_t)P;
        }
    });
}

// ---- SDFC v1 checkpoints (checkpoint.cpp:12-181) -----
// The on-disk tensors are little-endian f32, the device's own storage type,
// so a load is one parse + upload and a save one download + write;
// save(load(file)) reproduces the reference's bytes.
}  // extern "C"
namespace {
constexpr char kSdfcMagic[4] = {'S', 'D', 'F', 'C'};
constexpr uint32_t kSdfcVersion = 1;

struct SdfcWriter {
    FILE* f;
    const char* path;
    template <typename T> void pod(const T& v) {
        if (fwrite(&v, sizeof(T), 1, f) != 1) fail(PSDF_ERR_RUNTIME, "checkpoint: failed while writing: %s", path);
    }
    void tensor(const float* v, uint64_t n) {
        pod(n);
        if (n && fwrite(v, sizeof(float), n, f) != n) fail(PSDF_ERR_RUNTIME, "checkpoint: failed while writing: %s", path);
    }
};
struct SdfcReader {
    FILE* f;
    const char* path;
    template <typename T> void pod(T& v) {
        if (fread(&v, sizeof(T), 1, f) != 1) fail(PSDF_ERR_RUNTIME, "checkpoint: truncated file: %s", path);
    }
    void tensor(float* out, uint64_t expected) {
        uint64_t n = 0;
        pod(n);
        if (n != expected) fail(PSDF_ERR_RUNTIME, "checkpoint: tensor size mismatch in %s", path);
        if (n && fread(out, sizeof(float), n, f) != n) fail(PSDF_ERR_RUNTIME, "checkpoint: truncated file: %s", path);
    }
};
struct FileCloser {
    FILE* f;
    ~FileCloser() {
        if (f) fclose(f);
    }
};
}  // namespace
// ---- evaluation geometry: point-to-mesh distance and chamfer (metrics.cpp) --
// f64 with explicit round-to-nearest operations (no FMA contraction), in the
// reference's operation order, so every point-triangle distance is bit-equal
// to point_triangle_distance (metrics.cpp:11-47) compiled without contraction.
struct MV3 {
    double x, y, z;
};
__device__ __forceinline__ MV3 d3sub(MV3 a, MV3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ double d3dot(MV3 a, MV3 b) {  // Vec3::dot (vec.hpp:26)
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ MV3 d3axpy(MV3 a, MV3 d, double s) {  // a + d * s
    return {__dadd_rn(a.x, __dmul_rn(d.x, s)), __dadd_rn(a.y, __dmul_rn(d.y, s)), __dadd_rn(a.z, __dmul_rn(d.z, s))};
}
__device__ __forceinline__ double d3norm(MV3 a) { return __dsqrt_rn(d3dot(a, a)); }
__device__ __forceinline__ double dsub2(double a, double b, double c, double d) {  // a*b - c*d
    return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
}

// metrics.cpp:11-47 (Ericson's closest point on a triangle).
__device__ double point_triangle_distance(MV3 p, MV3 a, MV3 b, MV3 c) {
    const MV3 ab = d3sub(b, a), ac = d3sub(c, a), ap = d3sub(p, a);
    const double d1 = d3dot(ab, ap), d2 = d3dot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return d3norm(d3sub(p, a));
    const MV3 bp = d3sub(p, b);
    const double d3 = d3dot(ab, bp), d4 = d3dot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) return d3norm(d3sub(p, b));
    const double vc = dsub2(d1, d4, d3, d2);
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double v = __ddiv_rn(d1, __dsub_rn(d1, d3));
        return d3norm(d3sub(p, d3axpy(a, ab, v)));
    }
    const MV3 cp = d3sub(p, c);
    const double d5 = d3dot(ab, cp), d6 = d3dot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return d3norm(d3sub(p, c));
    const double vb = dsub2(d5, d2, d1, d6);
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = __ddiv_rn(d2, __dsub_rn(d2, d6));
        return d3norm(d3sub(p, d3axpy(a, ac, w)));
    }
    const double va = dsub2(d3, d6, d5, d4);
    const double e43 = __dsub_rn(d4, d3), e56 = __dsub_rn(d5, d6);
    if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
        const double w = __ddiv_rn(e43, __dadd_rn(e43, e56));
        return d3norm(d3sub(p, d3axpy(b, d3sub(c, b), w)));
    }
    const double denom = __ddiv_rn(1.0, __dadd_rn(__dadd_rn(va, vb), vc));
    const double v = __dmul_rn(vb, denom), w = __dmul_rn(vc, denom);
    return d3norm(d3sub(p, d3axpy(d3axpy(a, ab, v), ac, w)));
}

// Triangle soup (9 doubles per triangle) and one AABB per chunk of kTriChunk
// consecutive triangles (meshes from marching cubes are emitted cell by cell,
// so consecutive triangles are spatially coherent and the boxes are tight).
#ifndef PSDF_TRI_CHUNK
#define PSDF_TRI_CHUNK 64  // A/B 128 / 64 / 32 (profiles/r01/v19_eval_timing.log)
#endif
constexpr int kTriChunk = PSDF_TRI_CHUNK;
constexpr int kSeeds = 3;  // initial-bound chunks per block
__global__ void __launch_bounds__(kTriChunk) tri_soup_kernel(const double* __restrict__ verts, int64_t nv,
                                                             const int32_t* __restrict__ tris, int64_t nt,
                                                             double* __restrict__ soup, double* __restrict__ box,
                                                             unsigned long long* __restrict__ bad) {
    __shared__ double red[6][kTriChunk];
    const int64_t t = blockIdx.x * (int64_t)kTriChunk + threadIdx.x;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    if (t < nt) {
        for (int k = 0; k < 3; ++k) {
            int32_t vi = tris[3 * t + k];
            if (vi < 0 || vi >= nv) {
                atomicAdd(bad, 1ull);
                vi = 0;
            }
            for (int a = 0; a < 3; ++a) {
                const double x = verts[3 * (int64_t)vi + a];
                soup[9 * t + 3 * k + a] = x;
                lo[a] = fmin(lo[a], x);
                hi[a] = fmax(hi[a], x);
            }
        }
    }
    for (int a = 0; a < 3; ++a) {
        red[a][threadIdx.x] = lo[a];
        red[3 + a][threadIdx.x] = hi[a];
    }
    __syncthreads();
    for (int o = kTriChunk / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int a = 0; a < 3; ++a) {
                red[a][threadIdx.x] = fmin(red[a][threadIdx.x], red[a][threadIdx.x + o]);
                red[3 + a][threadIdx.x] = fmax(red[3 + a][threadIdx.x], red[3 + a][threadIdx.x + o]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) box[6 * blockIdx.x + threadIdx.x] = red[threadIdx.x][0];
}

// 30-bit Morton key of each point in the points' bounding box, so that a
// block's points are spatially coherent and its chunk culling is effective.
__global__ void __launch_bounds__(256) morton_kernel(const double* __restrict__ pts, int64_t n, double lx, double ly,
                                                     double lz, double inv, uint32_t* __restrict__ key,
                                                     int32_t* __restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto spread = [](double x) {
        uint32_t v = (uint32_t)fmin(fmax(x, 0.0), 1023.0);
        v = (v | (v << 16)) & 0x030000FFu;
        v = (v | (v << 8)) & 0x0300F00Fu;
        v = (v | (v << 4)) & 0x030C30C3u;
        v = (v | (v << 2)) & 0x09249249u;
        return v;
    };
    key[i] = (spread((pts[3 * i] - lx) * inv) << 2) | (spread((pts[3 * i + 1] - ly) * inv) << 1) |
             spread((pts[3 * i + 2] - lz) * inv);
    idx[i] = (int32_t)i;
}

__device__ __forceinline__ double box_dist(const double* bx, MV3 p) {  // metrics.cpp:104-110 shape
    const double dx = fmax(fmax(bx[0] - p.x, 0.0), p.x - bx[3]);
    const double dy = fmax(fmax(bx[1] - p.y, 0.0), p.y - bx[4]);
    const double dz = fmax(fmax(bx[2] - p.z, 0.0), p.z - bx[5]);
    return sqrt(dx * dx + dy * dy + dz * dz);
}

// Unsigned distance of each point to the mesh (MeshDistance::distance,
// metrics.cpp:131-135): the exact minimum over all triangles.  One thread per
// point, points in Morton order (perm); blockIdx.y splits the chunk range so
// the grid fills the GPU.  Each block first visits the chunks whose boxes are
// nearest its first, middle and last point (tight initial bounds), then every chunk of its
// range that some thread's point may be closer to than its current best
// (conservative margin, so the minimum is the brute-force one); chunks are
// staged in shared memory.  Partial minima meet in a u64 atomicMin on the
// f64 bit patterns (non-negative doubles order like their bits; out starts at
// all-ones).  NaN distances (degenerate triangles) never win, as with
// std::min(best, d).
#ifndef PSDF_PMD_MINB
#define PSDF_PMD_MINB 1
#endif
#ifndef PSDF_PMD_BLOCKS_PER_SM
#define PSDF_PMD_BLOCKS_PER_SM 16
#endif
__global__ void __launch_bounds__(kTriChunk, PSDF_PMD_MINB) point_mesh_distance_kernel(const double* __restrict__ pts, int64_t n,
                                                                        const int32_t* __restrict__ perm,
                                                                        const double* __restrict__ soup,
                                                                        const double* __restrict__ box, int64_t nt,
                                                                        unsigned long long* __restrict__ out) {
    __shared__ double tri[kTriChunk * 9];
    __shared__ double rd[kSeeds][kTriChunk];
    __shared__ int64_t ri[kSeeds][kTriChunk];
    const int64_t i = blockIdx.x * (int64_t)kTriChunk + threadIdx.x;
    const bool live = i < n;
    const int64_t pi = live ? perm[i] : 0;
    MV3 p = {0, 0, 0};
    if (live) p = {pts[3 * pi], pts[3 * pi + 1], pts[3 * pi + 2]};
    const int64_t nch = (nt + kTriChunk - 1) / kTriChunk;
    const int64_t c0 = nch * blockIdx.y / gridDim.y, c1 = nch * (blockIdx.y + 1) / gridDim.y;
    // seeds: the chunk box nearest the block's first, middle and last point
    // (a block's Morton range can straddle a code discontinuity)
    const int64_t blk0 = blockIdx.x * (int64_t)kTriChunk, nb = n - blk0 < kTriChunk ? n - blk0 : kTriChunk;
    MV3 q[kSeeds];
    double bd[kSeeds];
    int64_t bi[kSeeds];
#pragma unroll
    for (int j = 0; j < kSeeds; ++j) {
        const int64_t qi = perm[blk0 + (nb - 1) * j / (kSeeds - 1)];
        q[j] = {pts[3 * qi], pts[3 * qi + 1], pts[3 * qi + 2]};
        bd[j] = 1e300;
        bi[j] = 0;
    }
    for (int64_t ch = threadIdx.x; ch < nch; ch += kTriChunk)
#pragma unroll
        for (int j = 0; j < kSeeds; ++j) {
            const double d = box_dist(box + 6 * ch, q[j]);
            if (d < bd[j]) {
                bd[j] = d;
                bi[j] = ch;
            }
        }
#pragma unroll
    for (int j = 0; j < kSeeds; ++j) {
        rd[j][threadIdx.x] = bd[j];
        ri[j][threadIdx.x] = bi[j];
    }
    __syncthreads();
    for (int o = kTriChunk / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
#pragma unroll
            for (int j = 0; j < kSeeds; ++j) {
                const int t = threadIdx.x;
                if (rd[j][t + o] < rd[j][t] || (rd[j][t + o] == rd[j][t] && ri[j][t + o] < ri[j][t])) {
                    rd[j][t] = rd[j][t + o];
                    ri[j][t] = ri[j][t + o];
                }
            }
        __syncthreads();
    }
    int64_t seed[kSeeds];
#pragma unroll
    for (int j = 0; j < kSeeds; ++j) seed[j] = ri[j][0];
    double best = 1.7976931348623157e308;  // numeric_limits<double>::max()
    for (int64_t k = c0 - kSeeds; k < c1; ++k) {
        const bool is_seed = k < c0;
        int64_t ch = k;
        bool dup = false;
        if (is_seed) {
            const int j = (int)(k - (c0 - kSeeds));
            ch = seed[j];
            for (int jj = 0; jj < j; ++jj) dup |= seed[jj] == ch;
        } else {
            for (int jj = 0; jj < kSeeds; ++jj) dup |= seed[jj] == ch;
        }
        if (dup) continue;  // block-uniform
        const bool need = live && (is_seed || box_dist(box + 6 * ch, p) * (1.0 - 1e-9) <= best);
        if (!__syncthreads_or(need)) continue;
        const int64_t t0 = ch * kTriChunk;
        const int cnt = (int)(nt - t0 < kTriChunk ? nt - t0 : kTriChunk);
        for (int qq = threadIdx.x; qq < cnt * 9; qq += kTriChunk) tri[qq] = soup[9 * t0 + qq];
        __syncthreads();
        if (need)
            for (int qq = 0; qq < cnt; ++qq) {
                const double* v = tri + 9 * qq;
                best = fmin(best, point_triangle_distance(p, {v[0], v[1], v[2]}, {v[3], v[4], v[5]},
                                                          {v[6], v[7], v[8]}));
            }
        __syncthreads();
    }
    if (live) atomicMin(out + pi, (unsigned long long)__double_as_longlong(best));
}

// metrics.cpp:196-211 psnr_masked: squared error (three channels) over the
// pixels inside the mask, accumulated in f64 from the fp32 render; one f64 /
// u64 atomic pair per block.
__global__ void __launch_bounds__(256) psnr_partial_kernel(const float* __restrict__ rgb,
                                                           const float* __restrict__ gt,
                                                           const uint8_t* __restrict__ mask, int64_t px,
                                                           double* __restrict__ sq,
                                                           unsigned long long* __restrict__ n) {
    __shared__ double red[8];
    double s = 0.0;
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < px; i += (int64_t)gridDim.x * blockDim.x) {
        if (!mask[i]) continue;
        const double dx = (double)rgb[3 * i] - (double)gt[3 * i];
        const double dy = (double)rgb[3 * i + 1] - (double)gt[3 * i + 1];
        const double dz = (double)rgb[3 * i + 2] - (double)gt[3 * i + 2];
        s += (dx * dx + dy * dy) + dz * dz;  // Vec3::norm2
        cnt += 3;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n, cnt);
    block_add_f64(sq, s, red);
}

extern "C" {

int psdf_save_checkpoint(psdf_ctx* c, const char* path, int32_t lod, int32_t band_voxels, int32_t lod_cursor,
                         int64_t iteration, uint64_t seed) {
    return guarded([&] {
        need_grid(c);
        if (!path) fail(PSDF_ERR_INVALID_ARGUMENT, "null path");
        psdf_grid_desc d = c->desc;
        d.n_s = c->hns;  // the file holds the caller's widths
        d.n_a = c->hna;
        const int64_t T = d.T, P = d.P;
        const int64_t ps = 256 * d.n_s, pc = (int64_t)d.sh_order * d.sh_order * d.n_a;
        std::vector<int32_t> tc(3 * std::max<int64_t>(T, 1)), pco(3 * std::max<int64_t>(P, 1));
        std::vector<float> raw(T * TV), planes(T * 3 * ps), probes(P * pc), mlp(psdf_mlp_size(d.n_s, d.n_a, d.ncam));
        if (psdf_download_structure(c, tc.data(), nullptr, pco.data()) != PSDF_OK ||
            psdf_download_params(c, raw.data(), nullptr, planes.data(), probes.data(), mlp.data()) != PSDF_OK)
            fail(PSDF_ERR_RUNTIME, "%s", g_err.c_str());
        FileCloser fc{fopen(path, "wb")};
        if (!fc.f) fail(PSDF_ERR_RUNTIME, "checkpoint: cannot open for writing: %s", path);
        SdfcWriter w{fc.f, path};
        if (fwrite(kSdfcMagic, 1, 4, fc.f) != 4) fail(PSDF_ERR_RUNTIME, "checkpoint: failed while writing: %s", path);
        w.pod(kSdfcVersion);
        w.pod(d.voxel_size);
        for (int a = 0; a < 3; ++a) w.pod(d.origin[a]);
        w.pod(d.far_field_voxels);
        const int32_t ints[8] = {d.res[0], d.res[1], d.res[2], d.n_s, d.n_a, d.sh_order, lod, band_voxels};
        w.pod(ints);
        w.pod((uint32_t)T);
        for (int64_t t = 0; t < T; ++t) {
            const int32_t q[3] = {tc[3 * t], tc[3 * t + 1], tc[3 * t + 2]};
            w.pod(q);
        }
        for (int64_t t = 0; t < T; ++t) {
            w.tensor(raw.data() + t * TV, TV);
            for (int q = 0; q < 3; ++q) w.tensor(planes.data() + (t * 3 + q) * ps, ps);
        }
        w.pod((uint32_t)P);
        for (int64_t p = 0; p < P; ++p) {
            const int32_t q[3] = {pco[3 * p], pco[3 * p + 1], pco[3 * p + 2]};
            w.pod(q);
            w.tensor(probes.data() + p * pc, pc);
        }
        const MlpLayout G = MlpLayout::make(d.n_s + d.n_a + NPOW);
        const int32_t mints[3] = {d.n_s, d.n_a, d.ncam};
        w.pod(mints);
        w.tensor(mlp.data() + G.w1, G.b1 - G.w1);
        w.tensor(mlp.data() + G.b1, HID);
        w.tensor(mlp.data() + G.w2, HID * HID);
        w.tensor(mlp.data() + G.b2, HID);
        w.tensor(mlp.data() + G.w3, 3 * HID);
        w.tensor(mlp.data() + G.b3, 3);
        w.tensor(mlp.data() + G.cam, (uint64_t)d.ncam * HID);
        w.pod(lod_cursor);
        w.pod(iteration);
        w.pod(seed);
    });
}

int psdf_load_checkpoint(psdf_ctx* c, const char* path, int32_t* lod, int32_t* band_voxels, int32_t* lod_cursor,
                         int64_t* iteration, uint64_t* seed) {
    return guarded([&] {
        if (!c || !path) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        FileCloser fc{fopen(path, "rb")};
        if (!fc.f) fail(PSDF_ERR_RUNTIME, "checkpoint: cannot open: %s", path);
        SdfcReader r{fc.f, path};
        char magic[4];
        if (fread(magic, 1, 4, fc.f) != 4 || std::memcmp(magic, kSdfcMagic, 4) != 0)
            fail(PSDF_ERR_RUNTIME, "checkpoint: bad magic in %s", path);
        uint32_t version = 0;
        r.pod(version);
        if (version != kSdfcVersion) fail(PSDF_ERR_RUNTIME, "checkpoint: unsupported version %u in %s", version, path);
        psdf_grid_desc d{};
        r.pod(d.voxel_size);
        for (int a = 0; a < 3; ++a) r.pod(d.origin[a]);
        r.pod(d.far_field_voxels);
        int32_t ints[8];
        r.pod(ints);
        for (int a = 0; a < 3; ++a) d.res[a] = ints[a];
        d.n_s = ints[3];
        d.n_a = ints[4];
        d.sh_order = ints[5];
        if (d.sh_order < 1 || d.sh_order > 4 || d.n_s < 1 || d.n_a < 1)
            fail(PSDF_ERR_RUNTIME, "checkpoint: bad grid header in %s", path);
        uint32_t n_tiles = 0;
        r.pod(n_tiles);
        // tiles in file order; probes allocated corner by corner
        // (allocate_tile -> ensure_probe, grid.cpp:44-72)
        const int nt[3] = {d.res[0] / TE, d.res[1] / TE, d.res[2] / TE};
        std::vector<int32_t> tc(3 * (size_t)n_tiles), pid(8 * (size_t)n_tiles), pco;
        std::unordered_map<int64_t, int> probe_of;
        auto key = [&](int64_t x, int64_t y, int64_t z) { return (x * (nt[1] + 2) + y) * (nt[2] + 2) + z; };
        for (uint32_t t = 0; t < n_tiles; ++t) {
            int32_t q[3];
            r.pod(q);
            for (int a = 0; a < 3; ++a) tc[3 * t + a] = q[a];
            for (int i = 0; i < 8; ++i) {
                const int g[3] = {q[0] + (i & 1), q[1] + ((i >> 1) & 1), q[2] + ((i >> 2) & 1)};
                auto it = probe_of.find(key(g[0], g[1], g[2]));
                int id;
                if (it == probe_of.end()) {
                    id = (int)(pco.size() / 3);
                    probe_of.emplace(key(g[0], g[1], g[2]), id);
                    pco.insert(pco.end(), g, g + 3);
                } else {
                    id = it->second;
                }
                pid[8 * t + i] = id;
            }
        }
        const int64_t T = n_tiles, ps = 256 * (int64_t)d.n_s, pc = (int64_t)d.sh_order * d.sh_order * d.n_a;
        std::vector<float> raw(T * TV), planes(T * 3 * ps);
        for (int64_t t = 0; t < T; ++t) {
            r.tensor(raw.data() + t * TV, TV);
            for (int q = 0; q < 3; ++q) r.tensor(planes.data() + (t * 3 + q) * ps, ps);
        }
        uint32_t n_probes = 0;
        r.pod(n_probes);
        const int64_t P = (int64_t)(pco.size() / 3);
        if ((int64_t)n_probes != P) fail(PSDF_ERR_RUNTIME, "checkpoint: probe table inconsistent with tiles in %s", path);
        std::vector<float> probes(P * pc);
        for (uint32_t i = 0; i < n_probes; ++i) {
            int32_t q[3];
            r.pod(q);
            auto it = probe_of.find(key(q[0], q[1], q[2]));
            if (q[0] < 0 || q[1] < 0 || q[2] < 0 || it == probe_of.end())
                fail(PSDF_ERR_RUNTIME, "checkpoint: unknown probe coordinate in %s", path);
            r.tensor(probes.data() + (int64_t)it->second * pc, pc);
        }
        int32_t mints[3];
        r.pod(mints);
        if (mints[0] != d.n_s || mints[1] != d.n_a || mints[2] < 0)
            fail(PSDF_ERR_RUNTIME, "checkpoint: decoder does not match the grid's channels in %s", path);
        d.ncam = mints[2];
        const MlpLayout G = MlpLayout::make(d.n_s + d.n_a + NPOW);
        std::vector<float> mlp(psdf_mlp_size(d.n_s, d.n_a, d.ncam));
        r.tensor(mlp.data() + G.w1, G.b1 - G.w1);
        r.tensor(mlp.data() + G.b1, HID);
        r.tensor(mlp.data() + G.w2, HID * HID);
        r.tensor(mlp.data() + G.b2, HID);
        r.tensor(mlp.data() + G.w3, 3 * HID);
        r.tensor(mlp.data() + G.b3, 3);
        r.tensor(mlp.data() + G.cam, (uint64_t)d.ncam * HID);
        int32_t cursor = 0;
        int64_t iter = 0;
        uint64_t sd = 0;
        r.pod(cursor);
        r.pod(iter);
        r.pod(sd);
        d.T = (int)T;
        d.P = (int)P;
        if (psdf_upload_grid(c, &d, tc.data(), pid.data(), pco.data(), raw.data(), nullptr, planes.data(),
                             probes.data()) != PSDF_OK ||
            psdf_upload_mlp(c, mlp.data(), (int64_t)mlp.size()) != PSDF_OK)
            fail(PSDF_ERR_RUNTIME, "%s", g_err.c_str());
        if (lod) *lod = ints[6];
        if (band_voxels) *band_voxels = ints[7];
        if (lod_cursor) *lod_cursor = cursor;
        if (iteration) *iteration = iter;
        if (seed) *seed = sd;
    });
}

int psdf_set_keep_raypass_grads(psdf_ctx* c, int keep) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        c->keep_raypass = keep != 0;
        ensure_keep_buffers(c);
    });
}

int psdf_download_grads(psdf_ctx* c, int stage, float* raw, float* smooth, float* planes,
                        float* probes, float* mlp) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        if (stage != 0 && stage != 1) fail(PSDF_ERR_INVALID_ARGUMENT, "stage must be 0 or 1");
        if (stage == 0 && !c->keep_raypass)
            fail(PSDF_ERR_RUNTIME, "stage-0 gradients not kept (psdf_set_keep_raypass_grads)");
        const float* G = stage == 0 ? c->d_grads0 : c->d_grads;
        const float* S = stage == 0 ? c->d_gsmooth0 : c->d_gsmooth;
        download_params_host(c, G, S, raw, smooth, planes, probes, mlp);
    });
}

int psdf_smooth_all(psdf_ctx* c) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        c->last_launches = 0;
        smooth_all(c);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int psdf_render_device(psdf_ctx* c, const psdf_camera* cam, const psdf_render_opts* opt,
                       float* d_rgb, float* d_alpha, float* d_depth, psdf_counts* counts) {
    return guarded([&] {
        if (!d_rgb || !d_alpha) fail(PSDF_ERR_INVALID_ARGUMENT, "null output");
        do_render(c, cam, opt, d_rgb, d_alpha, d_depth, counts);
    });
}

int psdf_render(psdf_ctx* c, const psdf_camera* cam, const psdf_render_opts* opt, float* rgb,
                float* alpha, float* depth, psdf_counts* counts) {
    return guarded([&] {
        need_grid(c);
        if (!cam || !rgb || !alpha) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        check_camera(*cam);
        set_device(c);
        const size_t px = (size_t)cam->width * cam->height;
        ensure_dev(c->d_render, c->render_px, 5 * px);
        float* d_rgb = c->d_render;
        float* d_alpha = d_rgb + 3 * px;
        float* d_depth = depth ? d_alpha + px : nullptr;
        do_render(c, cam, opt, d_rgb, d_alpha, d_depth, counts);
        CK(cudaMemcpyAsync(rgb, d_rgb, sizeof(float) * 3 * px, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(alpha, d_alpha, sizeof(float) * px, cudaMemcpyDeviceToHost, c->stream));
        if (depth)
            CK(cudaMemcpyAsync(depth, d_depth, sizeof(float) * px, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int psdf_eval_psnr(psdf_ctx* c, const psdf_camera* cam, const psdf_render_opts* opt, const float* gt_rgb,
                   const uint8_t* mask, double* psnr, psdf_counts* counts) {
    return guarded([&] {
        need_grid(c);
        if (!cam || !gt_rgb || !mask || !psnr) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        check_camera(*cam);
        set_device(c);
        const size_t px = (size_t)cam->width * cam->height;
        // render scratch rgb | alpha | depth (unused) | gt rgb | mask bytes
        ensure_dev(c->d_render, c->render_px, 8 * px + px / 4 + 1);
        float* d_rgb = c->d_render;
        float* d_alpha = d_rgb + 3 * px;
        float* d_gt = d_rgb + 5 * px;
        uint8_t* d_mask = reinterpret_cast<uint8_t*>(d_rgb + 8 * px);
        CK(cudaMemcpyAsync(d_gt, gt_rgb, sizeof(float) * 3 * px, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_mask, mask, px, cudaMemcpyHostToDevice, c->stream));
        do_render(c, cam, opt, d_rgb, d_alpha, nullptr, counts);
        CK(cudaMemsetAsync(c->d_stats, 0, sizeof(double), c->stream));
        CK(cudaMemsetAsync(c->d_counts, 0, sizeof(unsigned long long), c->stream));
        const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(4 * c->sm_count, (int64_t)(px + 255) / 256));
        psnr_partial_kernel<<<blocks, 256, 0, c->stream>>>(d_rgb, d_gt, d_mask, (int64_t)px, c->d_stats,
                                                           c->d_counts);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_counts, c->d_counts, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const double sq = c->h_stats[0];
        const unsigned long long n = c->h_counts[0];
        double r = 99.0;
        if (n > 0) {
            const double mse = sq / (double)n;
            if (mse > 0.0) r = std::min(99.0, 10.0 * std::log10(1.0 / mse));
        }
        *psnr = r;
    });
}

// MeshDistance over a host mesh for host points (device-side distances).
static void mesh_distances(psdf_ctx* c, const double* pts, int64_t n, const double* verts, int64_t nv,
                           const int32_t* tris, int64_t nt, double* out) {
    if (nt <= 0) fail(PSDF_ERR_INVALID_ARGUMENT, "MeshDistance: empty mesh");  // metrics.cpp:49
    if (!verts || !tris || (n > 0 && (!pts || !out))) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
    if (nv <= 0) fail(PSDF_ERR_OUT_OF_RANGE, "triangle vertex index out of range");  // no vertex to index
    if (n == 0) return;
    if (n > INT32_MAX || nt > INT32_MAX) fail(PSDF_ERR_INVALID_ARGUMENT, "too many points or triangles");
    cudaStream_t s = c->stream;
    const int64_t nch = (nt + kTriChunk - 1) / kTriChunk;
    double lo[3] = {pts[0], pts[1], pts[2]}, hi[3] = {pts[0], pts[1], pts[2]};
    for (int64_t i = 1; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], pts[3 * i + a]);
            hi[a] = std::max(hi[a], pts[3 * i + a]);
        }
    const double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-300});
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                       (int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0, 30, s));
    // one grow-only arena: points | verts | soup | boxes | out | tris | keys | idx | sort temp
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t sz[9] = {al(24 * n), al(24 * nv), al(72 * nt), al(48 * nch), al(8 * n), al(12 * nt),
                          al(8 * n), al(8 * n), al(std::max<size_t>(tmp_bytes, 1))};
    size_t off[9], total = 0;
    for (int k = 0; k < 9; ++k) {
        off[k] = total;
        total += sz[k];
    }
    ensure_dev(c->d_eval, c->eval_cap, total);
    uint8_t* base = c->d_eval;
    double* d_pts = reinterpret_cast<double*>(base + off[0]);
    double* d_verts = reinterpret_cast<double*>(base + off[1]);
    double* d_soup = reinterpret_cast<double*>(base + off[2]);
    double* d_box = reinterpret_cast<double*>(base + off[3]);
    double* d_out = reinterpret_cast<double*>(base + off[4]);
    int32_t* d_tris = reinterpret_cast<int32_t*>(base + off[5]);
    uint32_t* d_key = reinterpret_cast<uint32_t*>(base + off[6]);
    int32_t* d_idx = reinterpret_cast<int32_t*>(base + off[7]);
    void* d_tmp = base + off[8];
    uint32_t* d_key2;
    int32_t* d_idx2;
    d_key2 = d_key + n;
    d_idx2 = d_idx + n;
    CK(cudaMemcpyAsync(d_pts, pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_verts, verts, sizeof(double) * 3 * nv, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_tris, tris, sizeof(int32_t) * 3 * nt, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(c->d_counts, 0, sizeof(unsigned long long), s));
    morton_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d_pts, n, lo[0], lo[1], lo[2], 1023.0 / ext, d_key,
                                                              d_idx);
    CK(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_key, d_key2, d_idx, d_idx2, (int)n, 0, 30, s));
    tri_soup_kernel<<<(unsigned)nch, kTriChunk, 0, s>>>(d_verts, nv, d_tris, nt, d_soup, d_box, c->d_counts);
    // split the chunk range over blockIdx.y until the grid holds ~16 blocks per SM
    const int64_t nblk = (n + kTriChunk - 1) / kTriChunk;
    const int64_t split = std::max<int64_t>(1, std::min<int64_t>({64, nch, (PSDF_PMD_BLOCKS_PER_SM * c->sm_count + nblk - 1) / nblk}));
    CK(cudaMemsetAsync(d_out, 0xff, sizeof(double) * n, s));
    point_mesh_distance_kernel<<<dim3((unsigned)nblk, (unsigned)split), kTriChunk, 0, s>>>(
        d_pts, n, d_idx2, d_soup, d_box, nt, reinterpret_cast<unsigned long long*>(d_out));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_counts, c->d_counts, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (c->h_counts[0]) fail(PSDF_ERR_OUT_OF_RANGE, "triangle vertex index out of range");
}

int psdf_point_mesh_distance(psdf_ctx* c, const double* points, int64_t n, const double* verts, int64_t nv,
                             const int32_t* tris, int64_t nt, double* out_dist) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        set_device(c);
        mesh_distances(c, points, n, verts, nv, tris, nt, out_dist);
    });
}

// directional_mean (metrics.cpp:168-179): summed on the host in point order
// from the device distances, so the mean is the reference's bit for bit.
static double directional_mean(const std::vector<double>& d, double max_dist) {
    double sum = 0.0;
    long count = 0;
    for (double x : d) {
        if (max_dist > 0.0 && x > max_dist) continue;
        sum += x;
        ++count;
    }
    return count > 0 ? sum / count : 0.0;
}

int psdf_chamfer(psdf_ctx* c, const double* pred_pts, int64_t n_pred, const double* pred_verts, int64_t pred_nv,
                 const int32_t* pred_tris, int64_t pred_nt, const double* gt_pts, int64_t n_gt,
                 const double* gt_verts, int64_t gt_nv, const int32_t* gt_tris, int64_t gt_nt, double max_dist,
                 double* out) {
    return guarded([&] {
        if (!c || !out) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        if (n_pred <= 0 || n_gt <= 0 || pred_nt <= 0 || gt_nt <= 0)  // metrics.cpp:185-186
            fail(PSDF_ERR_INVALID_ARGUMENT, "chamfer: empty input");
        set_device(c);
        std::vector<double> to_gt(n_pred), to_pred(n_gt);
        mesh_distances(c, pred_pts, n_pred, gt_verts, gt_nv, gt_tris, gt_nt, to_gt.data());
        mesh_distances(c, gt_pts, n_gt, pred_verts, pred_nv, pred_tris, pred_nt, to_pred.data());
        out[0] = 1000.0 * directional_mean(to_gt, max_dist);    // accuracy
        out[1] = 1000.0 * directional_mean(to_pred, max_dist);  // completeness
        out[2] = 0.5 * (out[0] + out[1]);
    });
}

// marching_cubes(grid) (mesh.cpp:363-394) of the context's smoothed SDF on the
// device (psdf_mesh.cuh); the mesh stays in the context for psdf_download_mesh.
int psdf_marching_cubes(psdf_ctx* c, int64_t* nv, int64_t* nt) {
    return guarded([&] {
        need_grid(c);
        if (!nv || !nt) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        set_device(c);
        cudaStream_t s = c->stream;
        const int64_t n = (int64_t)c->desc.T * TV;
        c->mesh_nv = c->mesh_nt = -1;
        if (n == 0) {
            c->mesh_nv = c->mesh_nt = 0;
            *nv = *nt = 0;
            return;
        }
        if (n > INT32_MAX) fail(PSDF_ERR_INVALID_ARGUMENT, "grid too large for marching cubes");
        size_t tmp_bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (int*)nullptr, (int*)nullptr, (int)n, s));
        auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
        const size_t o_own = al(2 * n), o_vc = o_own + al(2 * n), o_tc = o_vc + al(4 * n), o_tmp = o_tc + al(4 * n),
                     total = o_tmp + al(std::max<size_t>(tmp_bytes, 1));
        ensure_dev(c->d_mc, c->mc_cap, total);
        McView M{};
        M.g = c->view();
        M.cell = reinterpret_cast<uint16_t*>(c->d_mc);
        M.own = reinterpret_cast<uint16_t*>(c->d_mc + o_own);
        M.vcount = reinterpret_cast<int*>(c->d_mc + o_vc);
        M.tcount = reinterpret_cast<int*>(c->d_mc + o_tc);
        void* d_tmp = c->d_mc + o_tmp;
        for (int a = 0; a < 3; ++a) M.o[a] = c->desc.origin[a] + 0.5 * c->desc.voxel_size;  // voxel_center(0,0,0)
        const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 8 * c->sm_count);
        mc_case_kernel<<<blocks, 256, 0, s>>>(M);
        mc_own_kernel<<<blocks, 256, 0, s>>>(M);
        // vertex base per cell: exclusive scan of the owned-edge counts (in place)
        int last[2];
        CK(cudaMemcpyAsync(&last[0], M.vcount + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, M.vcount, M.vcount, (int)n, s));
        CK(cudaMemcpyAsync(&last[1], M.vcount + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t n_v = (int64_t)last[0] + last[1];
        // vertices first (the triangle pass reads them); triangles are counted,
        // scanned, and then the array is sized exactly
        ensure_dev(c->d_mesh, c->mesh_cap, al(24 * n_v) + 256);
        M.verts = reinterpret_cast<double*>(c->d_mesh);
        mc_vert_kernel<<<blocks, 256, 0, s>>>(M);
        mc_tri_kernel<false><<<blocks, 256, 0, s>>>(M);
        CK(cudaMemcpyAsync(&last[0], M.tcount + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, M.tcount, M.tcount, (int)n, s));
        CK(cudaMemcpyAsync(&last[1], M.tcount + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t n_t = (int64_t)last[0] + last[1];
        const size_t need = al(24 * n_v) + al(12 * n_t) + 256;
        if (need > c->mesh_cap) {  // grow, keeping the vertices
            uint8_t* p = nullptr;
            CK(cudaMalloc(&p, need));
            CK(cudaMemcpyAsync(p, c->d_mesh, 24 * n_v, cudaMemcpyDeviceToDevice, s));
            CK(cudaStreamSynchronize(s));
            cudaFree(c->d_mesh);
            c->d_mesh = p;
            c->mesh_cap = need;
            M.verts = reinterpret_cast<double*>(c->d_mesh);
        }
        M.tris = reinterpret_cast<int32_t*>(c->d_mesh + al(24 * n_v));
        mc_tri_kernel<true><<<blocks, 256, 0, s>>>(M);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        c->mesh_nv = n_v;
        c->mesh_nt = n_t;
        *nv = n_v;
        *nt = n_t;
    });
}

int psdf_download_mesh(psdf_ctx* c, double* verts, int32_t* tris) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        if (c->mesh_nv < 0) fail(PSDF_ERR_RUNTIME, "no mesh extracted (psdf_marching_cubes)");
        if ((c->mesh_nv > 0 && !verts) || (c->mesh_nt > 0 && !tris)) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        set_device(c);
        auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
        if (c->mesh_nv > 0)
            CK(cudaMemcpyAsync(verts, c->d_mesh, 24 * c->mesh_nv, cudaMemcpyDeviceToHost, c->stream));
        if (c->mesh_nt > 0)
            CK(cudaMemcpyAsync(tris, c->d_mesh + al(24 * c->mesh_nv), 12 * c->mesh_nt, cudaMemcpyDeviceToHost,
                               c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int psdf_train_reset(psdf_ctx* c) {
    return guarded([&] {
        need_grid(c);
        set_device(c);
        CK(cudaMemsetAsync(c->d_m, 0, sizeof(float) * c->n_params, c->stream));
        CK(cudaMemsetAsync(c->d_v, 0, sizeof(float) * c->n_params, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->adam_t = 0;
    });
}

int psdf_train_step(psdf_ctx* c, int n_views, const psdf_camera* cams, const float* const* gt_rgb,
                    const uint8_t* const* mask, const psdf_step_params* hp, psdf_losses* losses,
                    psdf_counts* counts) {
    return guarded([&] {
        need_grid(c);
        if (n_views <= 0 || !cams || !gt_rgb || !mask) fail(PSDF_ERR_INVALID_ARGUMENT, "empty batch");
        set_device(c);
        size_t px = 0;
        for (int i = 0; i < n_views; ++i) {
            check_camera(cams[i]);
            px += (size_t)cams[i].width * cams[i].height;
        }
        // stage this step's images into HBM (host -> device inside the step)
        size_t cap_rgb = c->stage_px * 3, cap_mask = c->stage_px;
        if (px > c->stage_px) {
            if (c->d_stage_rgb) cudaFree(c->d_stage_rgb);
            if (c->d_stage_mask) cudaFree(c->d_stage_mask);
            c->d_stage_rgb = nullptr;
            c->d_stage_mask = nullptr;
            cap_rgb = cap_mask = 0;
            ensure_dev(c->d_stage_rgb, cap_rgb, 3 * px);
            ensure_dev(c->d_stage_mask, cap_mask, px);
            c->stage_px = px;
        }
        std::vector<DevView> tmp(n_views);
        std::vector<DevView*> batch(n_views);
        // the pixel rows this rank's slice of the batch's 8x4 work tiles
        // covers (do_train_step: contiguous 1/N of the work tiles, each view's
        // tiles row-major): only those rows are copied, so the H2D bytes per
        // rank fall as 1/N; the staging buffer keeps the full layout
        std::vector<int> row0(n_views, 0), row1(n_views, -1);
        {
            int64_t tiles = 0;
            for (int i = 0; i < n_views; ++i)
                tiles += (int64_t)((cams[i].width + 7) / 8) * ((cams[i].height + 3) / 4);
            const int64_t tb = tiles * c->rank / c->world, te = tiles * (c->rank + 1) / c->world;
            int64_t begin = 0;
            for (int i = 0; i < n_views; ++i) {
                const int64_t tx = (cams[i].width + 7) / 8, n_t = tx * ((cams[i].height + 3) / 4);
                const int64_t lo = std::max(tb, begin), hi = std::min(te, begin + n_t);
                if (hi > lo) {
                    row0[i] = (int)(4 * ((lo - begin) / tx));
                    row1[i] = (int)std::min<int64_t>(cams[i].height - 1, 4 * ((hi - 1 - begin) / tx) + 3);
                }
                begin += n_t;
            }
        }
        size_t off = 0;
        CK(cudaStreamWaitEvent(c->copy_stream, c->ev_copy_free, 0));  // staging no longer read
        // masks first (the composite pass needs them), then the colours (the
        // photo terms); the scan reads neither and runs under the copies
        c->last_h2d_bytes = 0;
        for (int i = 0; i < n_views; ++i) {
            const size_t n = (size_t)cams[i].width * cams[i].height;
            tmp[i].cam = cams[i];
            tmp[i].rgb = c->d_stage_rgb + 3 * off;
            tmp[i].mask = c->d_stage_mask + off;
            batch[i] = &tmp[i];
            off += n;
            if (row1[i] < row0[i]) continue;
            const size_t o = (size_t)row0[i] * cams[i].width, m = (size_t)(row1[i] - row0[i] + 1) * cams[i].width;
            CK(cudaMemcpyAsync(tmp[i].mask + o, mask[i] + o, m, cudaMemcpyHostToDevice, c->copy_stream));
            c->last_h2d_bytes += (int64_t)m;
        }
        CK(cudaEventRecord(c->ev_masks, c->copy_stream));
        // the colours are read only at in-mask pixels (photo_pixel,
        // losses.cpp:8-38): only the rows between a view's first and last
        // row holding a mask pixel are copied.  The GPU finds those rows in
        // the copied masks (mask_rows_kernel on the copy stream, 8 bytes per
        // view back to pinned memory); the colour copies are enqueued from
        // inside the ray pass once its forward kernels are queued (the host
        // waits for the row extents there, long ready, while the GPU marches)
        if (n_views > c->rows_cap) {
            if (c->d_rows) cudaFree(c->d_rows);
            if (c->h_rows) cudaFreeHost(c->h_rows);
            c->d_rows = nullptr;
            c->h_rows = nullptr;
            c->rows_cap = 0;
            CK(cudaMalloc(&c->d_rows, sizeof(int) * 2 * n_views));
            CK(cudaMallocHost(&c->h_rows, sizeof(int) * 2 * n_views));
            c->rows_cap = n_views;
        }
        CK(cudaMemsetAsync(c->d_rows, 0xff, sizeof(int) * 2 * n_views, c->copy_stream));
        for (int i = 0; i < n_views; ++i) {
            if (row1[i] < row0[i]) continue;
            const int nr = row1[i] - row0[i] + 1;
            mask_rows_kernel<<<(unsigned)std::min(c->sm_count, (nr + 7) / 8), 256, 0, c->copy_stream>>>(
                tmp[i].mask, cams[i].width, row0[i], row1[i], c->d_rows + 2 * i);
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(c->h_rows, c->d_rows, sizeof(int) * 2 * n_views, cudaMemcpyDeviceToHost,
                           c->copy_stream));
        CK(cudaEventRecord(c->ev_rows, c->copy_stream));
        c->rgb_copy = [&, n_views]() {
            CK(cudaEventSynchronize(c->ev_rows));
            for (int i = 0; i < n_views; ++i) {
                const int m0 = c->h_rows[2 * i], m1 = c->h_rows[2 * i + 1];
                if (m0 < 0 || m1 < m0) continue;  // no mask pixel in the rank's rows
                const int w = cams[i].width;
                const size_t o = (size_t)m0 * w, m = (size_t)(m1 - m0 + 1) * w;
                CK(cudaMemcpyAsync(tmp[i].rgb + 3 * o, gt_rgb[i] + 3 * o, sizeof(float) * 3 * m,
                                   cudaMemcpyHostToDevice, c->copy_stream));
                c->last_h2d_bytes += (int64_t)(sizeof(float) * 3 * m);
            }
            CK(cudaEventRecord(c->ev_rgb, c->copy_stream));
            CK(cudaEventRecord(c->ev_copied, c->copy_stream));
        };
        c->images_pending = true;
        try {
            do_train_step(c, batch, hp, losses, counts, nullptr);
            // normally run by the ray pass; if not, the copies are issued now
            // and must land before the caller's buffers are released
            if (run_rgb_copy(c)) CK(cudaStreamSynchronize(c->copy_stream));
        } catch (...) {
            c->images_pending = false;
            if (c->rgb_copy) {  // keep ev_copied ordered after the masks at least
                c->rgb_copy = nullptr;
                cudaEventRecord(c->ev_rgb, c->copy_stream);
                cudaEventRecord(c->ev_copied, c->copy_stream);
            }
            cudaStreamSynchronize(c->copy_stream);  // no copy may outlive the call
            throw;
        }
        c->images_pending = false;
        CK(cudaStreamWaitEvent(c->stream, c->ev_copied, 0));
        CK(cudaEventRecord(c->ev_copy_free, c->stream));
        tmp.clear();
    });
}

int psdf_upload_views(psdf_ctx* c, int n_views, const psdf_camera* cams, const float* const* gt_rgb,
                      const uint8_t* const* mask) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        if (n_views < 0 || (n_views > 0 && (!cams || !gt_rgb || !mask)))
            fail(PSDF_ERR_INVALID_ARGUMENT, "bad view arrays");
        set_device(c);
        for (auto& v : c->views) {
            if (v.rgb) cudaFree(v.rgb);
            if (v.mask) cudaFree(v.mask);
        }
        c->views.assign(n_views, DevView{});
        for (int i = 0; i < n_views; ++i) {
            check_camera(cams[i]);
            const size_t n = (size_t)cams[i].width * cams[i].height;
            c->views[i].cam = cams[i];
            CK(cudaMalloc(&c->views[i].rgb, sizeof(float) * 3 * n));
            CK(cudaMalloc(&c->views[i].mask, n));
            CK(cudaMemcpyAsync(c->views[i].rgb, gt_rgb[i], sizeof(float) * 3 * n, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(c->views[i].mask, mask[i], n, cudaMemcpyHostToDevice, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
    });
}

int psdf_train_step_views(psdf_ctx* c, int n_batch, const int32_t* view_ids,
                          const psdf_step_params* hp, psdf_losses* losses, psdf_counts* counts) {
    return guarded([&] {
        need_grid(c);
        if (n_batch <= 0 || !view_ids) fail(PSDF_ERR_INVALID_ARGUMENT, "empty batch");
        std::vector<DevView*> batch(n_batch);
        for (int i = 0; i < n_batch; ++i) {
            if (view_ids[i] < 0 || view_ids[i] >= (int)c->views.size())
                fail(PSDF_ERR_OUT_OF_RANGE, "view id %d out of range", view_ids[i]);
            batch[i] = &c->views[view_ids[i]];
        }
        do_train_step(c, batch, hp, losses, counts);
    });
}

int psdf_debug_set_shard(psdf_ctx* c, int rank, int world_size) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        if (c->comm) fail(PSDF_ERR_RUNTIME, "context has a communicator");
        if (world_size < 1 || rank < 0 || rank >= world_size)
            fail(PSDF_ERR_INVALID_ARGUMENT, "bad rank %d / world %d", rank, world_size);
        c->rank = rank;
        c->world = world_size;
    });
}

// Diagnostics: raw copies of the last ray pass's queues (which: 0 e_slot i32,
// 1 e_acc f64, 2 e_craw f64x3, 3 e_nlive i32, 4 e_cfirst i32, 5 e_tfirst f64,
// 6 r_pos f64x3, 7 r_w f64, 8 r_tile i32, 9 r_entry i32, 10 a_t f64x2,
// 11 a_s f64x3, 12 a_i i32x4, 13 e_head i32, 14 e_ahead i32, 15 r_next i32).
int psdf_debug_wave(psdf_ctx* c, int which, void* out, int64_t n) {
    return guarded([&] {
        if (!c || !out) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        const WaveBufs& W = c->wave;
        const void* src = nullptr;
        size_t es = 0;
        switch (which) {
            case 0: src = W.e_slot; es = 4; break;
            case 1: src = W.e_acc; es = 8; break;
            case 2: src = W.e_craw; es = 24; break;
            case 3: src = W.e_nlive; es = 4; break;
            case 4: src = W.e_cfirst; es = 4; break;
            case 5: src = W.e_tfirst; es = 8; break;
            case 6: src = W.r_pos; es = 24; break;
            case 7: src = W.r_w; es = 8; break;
            case 8: src = W.r_tile; es = 4; break;
            case 9: src = W.r_entry; es = 4; break;
            case 10: src = W.a_t; es = 16; break;
            case 11: src = W.a_s; es = 24; break;
            case 12: src = W.a_i; es = 16; break;
            case 13: src = W.e_head; es = 4; break;
            case 14: src = W.e_ahead; es = 4; break;
            case 15: src = W.r_next; es = 4; break;
            default: fail(PSDF_ERR_INVALID_ARGUMENT, "bad queue %d", which);
        }
        if (!src) fail(PSDF_ERR_RUNTIME, "no ray pass yet");
        set_device(c);
        CK(cudaMemcpy(out, src, es * (size_t)n, cudaMemcpyDeviceToHost));
    });
}

int psdf_comm_unique_id(void* out) {
    return guarded([&] {
        if (!out) fail(PSDF_ERR_INVALID_ARGUMENT, "null output");
        g_nccl.load();
        ncclUniqueId id;
        NK(g_nccl.GetUniqueId(&id));
        static_assert(sizeof(ncclUniqueId) == PSDF_UNIQUE_ID_BYTES, "unique id size");
        std::memcpy(out, &id, sizeof id);
    });
}

int psdf_comm_init(psdf_ctx* c, const void* unique_id, int rank, int world_size) {
    return guarded([&] {
        if (!c || !unique_id) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        if (world_size < 1 || rank < 0 || rank >= world_size)
            fail(PSDF_ERR_INVALID_ARGUMENT, "bad rank %d / world %d", rank, world_size);
        set_device(c);
        c->rank = rank;
        c->world = world_size;
        // a single rank has nothing to exchange — unless PSDF_FORCE_NCCL asks
        // for the communicator anyway (tests: the NCCL path on one GPU)
        if (world_size == 1 && !std::getenv("PSDF_FORCE_NCCL")) return;
        g_nccl.load();
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof id);
        NK(g_nccl.CommInitRank(&c->comm, world_size, id, rank));
    });
}

int psdf_set_grad_exchange(psdf_ctx* c, int mode) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        if (mode < PSDF_EXCHANGE_ALLREDUCE || mode > PSDF_EXCHANGE_SHARDED)
            fail(PSDF_ERR_INVALID_ARGUMENT, "unknown gradient exchange %d", mode);
        set_device(c);
        c->grad_exchange = mode;
        if (mode == PSDF_EXCHANGE_BUCKETED && !c->comm_stream) {
            CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->ev_bucket, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_bucket_done, cudaEventDisableTiming));
        }
    });
}

int psdf_march_rays(psdf_ctx* c, int n, const double* origins, const double* dirs, int n_max,
                    double* ts, int32_t* counts) {
    return guarded([&] {
        need_grid(c);
        if (n < 0 || n_max < 0 || (n > 0 && (!origins || !dirs || !ts || !counts)))
            fail(PSDF_ERR_INVALID_ARGUMENT, "bad march arguments");
        if (n == 0) return;
        set_device(c);
        const int nm = std::max(n_max, 1);
        DevScratch scratch;
        double* d_o = scratch.alloc<double>((size_t)3 * n);
        double* d_d = scratch.alloc<double>((size_t)3 * n);
        double* d_t = scratch.alloc<double>((size_t)n * nm);
        int* d_n = scratch.alloc<int>((size_t)n);
        CK(cudaMemcpyAsync(d_o, origins, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_d, dirs, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        march_rays_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(c->view(), n, d_o, d_d, n_max, d_t, d_n);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMemcpyAsync(ts, d_t, sizeof(double) * (size_t)n * nm, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(counts, d_n, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int psdf_pixel_dirs(const psdf_camera* cam, double* out) {
    return guarded([&] {
        if (!cam || !out) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        check_camera(*cam);
        const int n = cam->width * cam->height;
        double* d;
        CK(cudaMalloc(&d, sizeof(double) * 3 * n));
        pixel_dirs_kernel<<<(n + 127) / 128, 128>>>(to_cam(*cam), d);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, d, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
        cudaFree(d);
    });
}

int psdf_last_k2_breakdown(psdf_ctx* c, double* ms4, int64_t* entries, int64_t* records) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        for (int k = 0; k < 4; ++k)
            if (ms4) ms4[k] = c->last_k2_ms[k];
        if (entries) *entries = c->last_entries;
        if (records) *records = c->last_records;
    });
}

int psdf_last_wave_counts(psdf_ctx* c, int64_t* out5) {
    return guarded([&] {
        if (!c || !out5) fail(PSDF_ERR_INVALID_ARGUMENT, "null argument");
        for (int k = 0; k < 5; ++k) out5[k] = c->last_wave[k];
    });
}

int psdf_last_timing(psdf_ctx* c, double* ray_ms, double* step_ms, int* launches) {
    return guarded([&] {
        if (!c) fail(PSDF_ERR_INVALID_ARGUMENT, "null context");
        if (ray_ms) *ray_ms = c->last_ray_ms;
        if (step_ms) *step_ms = c->last_step_ms;
        if (launches) *launches = c->last_launches;
    });
}

void* psdf_stream(psdf_ctx* c) { return c ? (void*)c->stream : nullptr; }

int64_t psdf_last_h2d_bytes(psdf_ctx* c) { return c ? c->last_h2d_bytes : -1; }

void* psdf_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void psdf_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
