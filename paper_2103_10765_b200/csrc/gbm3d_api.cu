// C ABI of libgbm3d.so (include/gbm3d.h): argument validation, grid geometry, kernel dispatch.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../include/gbm3d.h"
#include "common.cuh"
#include "match_direct.cuh"
#include "match_strip.cuh"
#include "strip_p8s8.cuh"
#include "strip_p12s4.cuh"
#include "match_tc16.cuh"
#include "match_tcp.cuh"

namespace gbm3d {

static thread_local int g_last_launches = 0;

// Fast-path table: (patch, stride) pairs with an instantiated strip kernel.  Heap depth by K
// (15 / 31 / 63 slots), key shift CB by radius (11 for r <= 22, 13 up to 32).
template <int PP, int SS, int TRY, int D, int WPS>
static cudaError_t launch_shape(const MatchParams& p, cudaStream_t st, int* launches) {
    const int L = p.K - 1;
    if (p.cb == 11) {
        if (L <= 15) return launch_strip<StripCfg<PP, SS, TRY, D, 11, WPS, 3>>(p, st, launches);
        if (L <= 31) return launch_strip<StripCfg<PP, SS, TRY, D, 11, WPS, 4>>(p, st, launches);
        return launch_strip<StripCfg<PP, SS, TRY, D, 11, WPS, 5>>(p, st, launches);
    }
    if (L <= 15) return launch_strip<StripCfg<PP, SS, TRY, D, 13, WPS, 3>>(p, st, launches);
    if (L <= 31) return launch_strip<StripCfg<PP, SS, TRY, D, 13, WPS, 4>>(p, st, launches);
    return launch_strip<StripCfg<PP, SS, TRY, D, 13, WPS, 5>>(p, st, launches);
}

static cudaError_t strip_dispatch(const MatchParams& p, cudaStream_t st, int* launches, bool* ok) {
    *ok = true;
    switch (p.P * 100 + p.S) {
        case 803: return launch_shape<8, 3, 4, 8, 1>(p, st, launches);     // solo warps
        case 1204: return launch_shape<12, 4, GBM3D_S12_TRY, GBM3D_S12_D, GBM3D_S12_WPS>(p, st, launches);
        case 802: return launch_shape<8, 2, 8, 5, 2>(p, st, launches);
        case 804: return launch_shape<8, 4, 6, 4, 2>(p, st, launches);
        case 808: return launch_shape<8, 8, GBM3D_S8_TRY, GBM3D_S8_D, GBM3D_S8_WPS>(p, st, launches);  // stage-1 tiling
        default: *ok = false; return cudaSuccess;
    }
}

// Tensor-core product-form kernels: patch 8, stride 3, the tile's candidate columns
// 7S + 2r + 1 <= 64 (radius <= 21), 2 <= K <= 32.  PRODUCT = fp16 kernel (match_tc16.cuh) with
// the exact int8 kernel (match_tc.cuh) redoing tiles outside the fp16 range bound;
// PRODUCT_I8 = the int8 kernel alone.
extern template cudaError_t launch_tc<3, 15>(const MatchParams&, cudaStream_t, int*, int);
extern template cudaError_t launch_tc<3, 31>(const MatchParams&, cudaStream_t, int*, int);
extern template cudaError_t launch_tc16<3, 15>(const MatchParams&, cudaStream_t, int*);
extern template cudaError_t launch_tc16<3, 31>(const MatchParams&, cudaStream_t, int*);
extern template cudaError_t launch_tcp<12, 4, 15, 64>(const MatchParams&, cudaStream_t, int*);
extern template cudaError_t launch_tcp<12, 4, 31, 64>(const MatchParams&, cudaStream_t, int*);
extern template cudaError_t launch_tcp<12, 4, 15, 80>(const MatchParams&, cudaStream_t, int*);
extern template cudaError_t launch_tcp<12, 4, 31, 80>(const MatchParams&, cudaStream_t, int*);
static cudaError_t tc_dispatch(const MatchParams& p, cudaStream_t st, int* launches, bool* ok,
                               bool int8_only) {
    *ok = false;
    // patch 12 / stride 4 (c2): fp16 product form with in-kernel exact paths (tiles above the
    // fp16 bound; references whose 32-bit-key lists end short when tau - 1 > dsat); the tile's
    // columns within N: 16 x 7 tiles when 6S + 2r + 1 <= 64, else 16 x 8 tiles with
    // 7S + 2r + 1 <= 80 (radius <= 21, the shared-memory bound)
    if (p.P == 12 && p.S == 4 && !int8_only && p.r <= tcp::MAX_R && 7 * p.S + 2 * p.r + 1 <= 80 &&
        p.K >= 2 && p.K <= 32) {
        *ok = true;
        if (6 * p.S + 2 * p.r + 1 <= 64) {
            if (p.K - 1 <= 15) return launch_tcp<12, 4, 15, 64>(p, st, launches);
            return launch_tcp<12, 4, 31, 64>(p, st, launches);
        }
        if (p.K - 1 <= 15) return launch_tcp<12, 4, 15, 80>(p, st, launches);
        return launch_tcp<12, 4, 31, 80>(p, st, launches);
    }
    if (p.P != 8 || p.S != 3 || 7 * p.S + 2 * p.r + 1 > tcm::NB || p.K < 2 || p.K > 32)
        return cudaSuccess;
    *ok = true;
    if (int8_only) {
        if (p.K - 1 <= 15) return launch_tc<3, 15>(p, st, launches, 0);
        return launch_tc<3, 31>(p, st, launches, 0);
    }
    if (p.K - 1 <= 15) return launch_tc16<3, 15>(p, st, launches);
    return launch_tc16<3, 31>(p, st, launches);
}

static int grid_count(int L, int P, int S) { return (L - P) / S + 1 + (((L - P) % S) ? 1 : 0); }

// Validate and fill the launch parameters shared by every entry point.
static int make_params(MatchParams& p, int B, int H, int W, int patch, int stride, int radius,
                       int K, int64_t tau) {
    if (B < 1 || H < 1 || W < 1 || patch < 1 || stride < 1 || radius < 0 || K < 1 || tau < 0)
        return GBM3D_ERR_ARG;
    if (H < patch || W < patch) return GBM3D_ERR_ARG;
    if ((long long)H * (long long)W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if (patch > 16 || radius > 32 || K > 64) return GBM3D_ERR_UNSUPPORTED;
    p = MatchParams{};
    p.B = B;
    p.H = H;
    p.W = W;
    p.P = patch;
    p.S = stride;
    p.r = radius;
    p.K = K;
    p.tau = tau;
    p.Ry = grid_count(H, patch, stride);
    p.Rx = grid_count(W, patch, stride);
    p.Ry_reg = (H - patch) / stride + 1;
    p.Rx_reg = (W - patch) / stride + 1;
    p.img_bstride = (int64_t)H * W;
    p.out_bstride = (int64_t)p.Ry * p.Rx;
    p.slab_y0 = 0;
    p.slab_y1 = H;
    p.row_begin = 0;
    p.row_end = p.Ry;
    p.side = 2 * radius + 1;
    // key = d << cb | code with 2^cb > side^2: cb = 11 for radius <= 22, 13 up to radius 32
    p.cb = ((long long)p.side * p.side < 2048) ? 11 : 13;
    p.dsat = (uint32_t)((1ULL << (32 - p.cb)) - 1ULL);
    const int64_t taum1 = tau - 1;  // strict: d < tau  <=>  d <= tau - 1
    p.tdr0 = (int)(taum1 < (int64_t)p.dsat ? taum1 : (int64_t)p.dsat);
    p.thr0 = (tau <= (int64_t)p.dsat) ? (uint32_t)((uint64_t)tau << p.cb) : KEY_INF;
    p.tau_above_dsat = taum1 > (int64_t)p.dsat ? 1 : 0;
    return GBM3D_OK;
}

static cudaError_t launch_direct(const MatchParams& p, cudaStream_t st, int k_begin, int k_end,
                                 int m_begin, int m_end, int* launches) {
    if (k_end <= k_begin || m_end <= m_begin) return cudaSuccess;
    // compile-time patch for the common shapes (unrolled rows), any P <= 16 otherwise
    auto kern = p.P == 8 ? match_direct_kernel<8> : p.P == 12 ? match_direct_kernel<12>
              : p.P == 16 ? match_direct_kernel<16> : match_direct_kernel<0>;
    const long long nref = (long long)(k_end - k_begin) * (m_end - m_begin);
    dim3 grid((unsigned)nref, 1, p.B);
    // one thread per task of 8 candidates of a full window (rounded to warps, 64..256): no
    // idle warps for small windows (P16 r16: 33 x 5 tasks -> 192 threads)
    const int side = 2 * p.r + 1, ntask = side * ((side + DIRECT_CG - 1) / DIRECT_CG);
    const int nthr = std::max(64, std::min(DIRECT_THREADS, (ntask + 31) / 32 * 32));
    kern<<<grid, nthr, 0, st>>>(p, k_begin, m_begin, m_end - m_begin);
    if (launches) ++*launches;
    return cudaGetLastError();
}

// Dispatch one call: strip kernel over the regular grid part, direct kernel for the appended
// row/column (reading R3), or direct for everything when no fast kernel fits.
// GBM3D_DEBUG=1 prints the CUDA error behind a GBM3D_ERR_CUDA status (stderr).
static int cuda_fail(cudaError_t e, const char* where) {
    static const bool dbg = getenv("GBM3D_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "gbm3d: %s: %s\n", where, cudaGetErrorString(e));
    return GBM3D_ERR_CUDA;
}

// Two library-owned side streams per host thread for the direct kernel's appended row and
// column: they depend only on the inputs, so they fork from the caller's stream before the
// fast kernel and join after it (the three run concurrently; capturable in CUDA graphs).
struct SideStreams {
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
    bool ok = false, tried = false;
    bool init() {
        if (tried) return ok;
        tried = true;
        for (int i = 0; i < 2; ++i) {
            if (cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking) != cudaSuccess) return false;
            if (cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming) != cudaSuccess) return false;
        }
        if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return false;
        ok = true;
        return true;
    }
};
// one set per (host thread, device): library streams belong to the device current at creation
constexpr int kMaxDevices = 16;
static thread_local SideStreams g_side_dev[kMaxDevices];
static SideStreams* side_for_current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    SideStreams* sd = &g_side_dev[dev];
    return sd->init() ? sd : nullptr;
}

// AUTO on tiny jobs (latency cases): the tile kernels need about one tile's time on
// one SM however few references there are (c0: 68 us), while the per-reference direct kernel
// spreads the references over every SM (c0: 26 us).  Below this much pixel work (references x
// window x patch^2) the direct kernel is faster (c0 3.9e7: direct; c1 6.9e8: tile kernels).
// GBM3D_NO_SMALL_DIRECT=1 turns the rule off (the parity tests keep the tile kernels on their
// small edge-case images).
constexpr double kSmallDirectWork = 1.2e8;
static bool small_direct(const MatchParams& p) {
    static const bool off = getenv("GBM3D_NO_SMALL_DIRECT") != nullptr;
    if (off) return false;
    const double side = 2.0 * p.r + 1.0;
    const double work = (double)p.B * (double)(p.row_end - p.row_begin) * (double)p.Rx * side * side *
                        (double)p.P * (double)p.P;
    return work < kSmallDirectWork;
}

static int run(const MatchParams& p, int method, cudaStream_t st) {
    int launches = 0;
    cudaError_t e = cudaSuccess;
    bool fast = false;
    if (method == GBM3D_METHOD_AUTO && small_direct(p)) method = GBM3D_METHOD_DIRECT;
    const int kr1_ = std::min(p.row_end, p.Ry_reg);
    const bool app_col = p.Rx > p.Rx_reg && kr1_ > p.row_begin;
    const bool app_row = p.Ry > p.Ry_reg && p.row_end > p.Ry_reg;
    SideStreams* const sd =
        (method != GBM3D_METHOD_DIRECT && (app_col || app_row)) ? side_for_current_device() : nullptr;
    const bool side = sd != nullptr;
    if (side && cudaEventRecord(sd->fork, st) != cudaSuccess) return cuda_fail(cudaGetLastError(), "fork");
    if (method == GBM3D_METHOD_AUTO || method == GBM3D_METHOD_PRODUCT ||
        method == GBM3D_METHOD_PRODUCT_I8) {
        // AUTO prefers the tensor-core product form (fastest where it applies)
        e = tc_dispatch(p, st, &launches, &fast, method == GBM3D_METHOD_PRODUCT_I8);
        if (e != cudaSuccess) return cuda_fail(e, "tensor-core kernels");
        if (!fast && method != GBM3D_METHOD_AUTO) return GBM3D_ERR_UNSUPPORTED;
    }
    if (!fast && (method == GBM3D_METHOD_AUTO || method == GBM3D_METHOD_SSD)) {
        e = strip_dispatch(p, st, &launches, &fast);
        if (e != cudaSuccess) return cuda_fail(e, "strip kernel");
        if (!fast && method == GBM3D_METHOD_SSD) return GBM3D_ERR_UNSUPPORTED;
    }
    if (fast) {
        const int kr1 = kr1_;
        // appended column for the regular rows of the call, appended row (all columns) when it
        // is inside the call's row range: on the side streams when available
        cudaStream_t sc = side ? sd->s[0] : st, sr = side ? sd->s[1] : st;
        if (app_col) {
            if (side && cudaStreamWaitEvent(sc, sd->fork, 0) != cudaSuccess) return GBM3D_ERR_CUDA;
            e = launch_direct(p, sc, p.row_begin, kr1, p.Rx_reg, p.Rx, &launches);
            if (e == cudaSuccess && side) e = cudaEventRecord(sd->join[0], sc);
            if (e == cudaSuccess && side) e = cudaStreamWaitEvent(st, sd->join[0], 0);
        }
        if (e == cudaSuccess && app_row) {
            if (side && cudaStreamWaitEvent(sr, sd->fork, 0) != cudaSuccess) return GBM3D_ERR_CUDA;
            e = launch_direct(p, sr, std::max(p.row_begin, p.Ry_reg), p.row_end, 0, p.Rx, &launches);
            if (e == cudaSuccess && side) e = cudaEventRecord(sd->join[1], sr);
            if (e == cudaSuccess && side) e = cudaStreamWaitEvent(st, sd->join[1], 0);
        }
    } else {
        e = launch_direct(p, st, p.row_begin, p.row_end, 0, p.Rx, &launches);
    }
    if (e != cudaSuccess) return GBM3D_ERR_CUDA;
    g_last_launches = launches;
    return GBM3D_OK;
}

// ---- range precondition (reading R10)
__global__ void range_minmax_kernel(const int16_t* __restrict__ img, int64_t n, int* out) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int v = img[i];
        lo = min(lo, v);
        hi = max(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

}  // namespace gbm3d

using namespace gbm3d;

extern "C" {

int gbm3d_grid_dims(int H, int W, int patch, int stride, int* n_ref_y, int* n_ref_x) {
    if (patch < 1 || stride < 1 || H < patch || W < patch) return GBM3D_ERR_ARG;
    if (n_ref_y) *n_ref_y = grid_count(H, patch, stride);
    if (n_ref_x) *n_ref_x = grid_count(W, patch, stride);
    return GBM3D_OK;
}

int gbm3d_block_match_ex(const int16_t* imgs, int B, int H, int W, int patch, int stride,
                         int radius, int K, int64_t tau, int method, int32_t* idx,
                         int32_t* dist, int32_t* n_valid, void* stream) {
    if (!imgs || !idx || !dist) return GBM3D_ERR_ARG;
    if (method < GBM3D_METHOD_AUTO || method > GBM3D_METHOD_PRODUCT_I8) return GBM3D_ERR_ARG;
    MatchParams p;
    const int st = make_params(p, B, H, W, patch, stride, radius, K, tau);
    if (st != GBM3D_OK) return st;
    p.img = imgs;
    p.idx = idx;
    p.dist = dist;
    p.nvalid = n_valid;
    return run(p, method, (cudaStream_t)stream);
}

int gbm3d_block_match(const int16_t* img, int H, int W, int patch, int stride, int radius, int K,
                      int64_t tau, int32_t* idx, int32_t* dist, int32_t* n_valid, void* stream) {
    return gbm3d_block_match_ex(img, 1, H, W, patch, stride, radius, K, tau, GBM3D_METHOD_AUTO,
                                idx, dist, n_valid, stream);
}

int gbm3d_block_match_batched(const int16_t* imgs, int B, int H, int W, int patch, int stride,
                              int radius, int K, int64_t tau, int32_t* idx, int32_t* dist,
                              int32_t* n_valid, void* stream) {
    return gbm3d_block_match_ex(imgs, B, H, W, patch, stride, radius, K, tau, GBM3D_METHOD_AUTO,
                                idx, dist, n_valid, stream);
}

int gbm3d_block_match_rows(const int16_t* slab, int slab_y0, int slab_rows, int H, int W,
                           int patch, int stride, int radius, int K, int64_t tau,
                           int ref_row_begin, int ref_row_end, int32_t* idx, int32_t* dist,
                           int32_t* n_valid, void* stream) {
    if (!slab || !idx || !dist) return GBM3D_ERR_ARG;
    MatchParams p;
    const int st = make_params(p, 1, H, W, patch, stride, radius, K, tau);
    if (st != GBM3D_OK) return st;
    if (ref_row_begin < 0 || ref_row_end > p.Ry || ref_row_begin >= ref_row_end)
        return GBM3D_ERR_ARG;
    if (slab_y0 < 0 || slab_rows < 1 || slab_y0 + slab_rows > H) return GBM3D_ERR_ARG;
    const int y_first = grid_pos(ref_row_begin, p.Ry_reg, stride, H - patch);
    const int y_last = grid_pos(ref_row_end - 1, p.Ry_reg, stride, H - patch);
    const int need0 = std::max(0, y_first - radius);
    const int need1 = std::min(H, y_last + radius + patch);
    if (slab_y0 > need0 || slab_y0 + slab_rows < need1) return GBM3D_ERR_ARG;
    p.img = slab;
    p.slab_y0 = slab_y0;
    p.slab_y1 = slab_y0 + slab_rows;
    p.row_begin = ref_row_begin;
    p.row_end = ref_row_end;
    p.idx = idx;
    p.dist = dist;
    p.nvalid = n_valid;
    p.out_bstride = (int64_t)(ref_row_end - ref_row_begin) * p.Rx;
    return run(p, GBM3D_METHOD_AUTO, (cudaStream_t)stream);
}

size_t gbm3d_host_workspace_bytes(int B, int H, int W, int patch, int stride, int K) {
    if (B < 1 || patch < 1 || stride < 1 || H < patch || W < patch || K < 1) return 0;
    const size_t img = ((size_t)B * H * W * 2 + 255) & ~(size_t)255;
    const size_t nref = (size_t)B * grid_count(H, patch, stride) * grid_count(W, patch, stride);
    const size_t tab = (nref * K * 4 + 255) & ~(size_t)255;
    const size_t nv = (nref * 4 + 255) & ~(size_t)255;
    return img + 2 * tab + nv;
}

// Host entry, pipelined: the job is cut into chunks (images for B > 1, blocks of reference
// rows for B = 1); the host-to-device copies run on one library stream, the matching of chunk
// c alternately on the caller's stream and a second compute stream (consecutive chunks may
// overlap on the SMs, so no chunk ends on a partial wave), and the device-to-host copies of
// chunk c on a third stream while later chunks are matched.  PCIe is full duplex, so
// the copies hide behind each other and behind the kernels.  The library streams and events
// are created once per host thread and device (thread_local) and reused; nothing else is
// allocated.
namespace {
constexpr int kMaxChunks = 64;
struct HostPipe {
    cudaStream_t h2d = nullptr, d2h = nullptr, comp2 = nullptr;
    cudaEvent_t in[kMaxChunks], done[kMaxChunks], out_done, start;
    bool ok = false;
    bool init() {
        if (ok) return true;
        if (cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) != cudaSuccess) return false;
        if (cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) != cudaSuccess) return false;
        if (cudaStreamCreateWithFlags(&comp2, cudaStreamNonBlocking) != cudaSuccess) return false;
        for (int i = 0; i < kMaxChunks; ++i) {
            if (cudaEventCreateWithFlags(&in[i], cudaEventDisableTiming) != cudaSuccess) return false;
            if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) return false;
        }
        if (cudaEventCreateWithFlags(&out_done, cudaEventDisableTiming) != cudaSuccess) return false;
        if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) != cudaSuccess) return false;
        ok = true;
        return true;
    }
};
thread_local HostPipe g_pipe_dev[kMaxDevices];
}  // namespace

int gbm3d_block_match_host(const int16_t* h_imgs, int B, int H, int W, int patch, int stride,
                           int radius, int K, int64_t tau, int32_t* h_idx, int32_t* h_dist,
                           int32_t* h_n_valid, void* d_workspace, size_t workspace_bytes,
                           void* stream) {
    if (!h_imgs || !h_idx || !h_dist || !d_workspace) return GBM3D_ERR_ARG;
    const size_t need = gbm3d_host_workspace_bytes(B, H, W, patch, stride, K);
    if (need == 0 || workspace_bytes < need) return GBM3D_ERR_ARG;
    MatchParams p;
    int st = make_params(p, B, H, W, patch, stride, radius, K, tau);
    if (st != GBM3D_OK) return st;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return GBM3D_ERR_CUDA;
    HostPipe& g_pipe = g_pipe_dev[dev];
    if (!g_pipe.init()) return GBM3D_ERR_CUDA;
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)d_workspace;
    const size_t img_b = (size_t)B * H * W * 2;
    const size_t per_img_refs = (size_t)p.Ry * p.Rx;
    const size_t nref = (size_t)B * per_img_refs;
    int16_t* d_img = (int16_t*)ws;
    int32_t* d_idx = (int32_t*)(ws + ((img_b + 255) & ~(size_t)255));
    int32_t* d_dist = (int32_t*)((char*)d_idx + ((nref * K * 4 + 255) & ~(size_t)255));
    int32_t* d_nv = (int32_t*)((char*)d_dist + ((nref * K * 4 + 255) & ~(size_t)255));
    // chunk plan: [ub[c], ub[c+1]) in images (B > 1) or in reference rows (B = 1, multiples of
    // 16 so the tensor-core tiles of a chunk are the tiles of the whole call; a short first
    // chunk so the copies out start early)
#ifndef GBM3D_HOST_NCH
#define GBM3D_HOST_NCH 16
#endif
    const int units = B > 1 ? B : p.Ry;
    int ub[kMaxChunks + 1];
    int nch = 0;
    if (B > 1) {
        const int n = std::min(B, GBM3D_HOST_NCH), step = (B + n - 1) / n;
        for (int u = 0; u < B; u += step) ub[nch++] = u;
    } else {
        const int first = std::min(units, 32);
        ub[nch++] = 0;
        if (first < units) {
            ub[nch++] = first;
            const int n = std::max(1, std::min(GBM3D_HOST_NCH - 1, (units - first) / 32));
            const int step = (((units - first + n - 1) / n) + 15) & ~15;
            for (int u = first + step; u < units; u += step) ub[nch++] = u;
        }
    }
    ub[nch] = units;
    if (nch > kMaxChunks) return GBM3D_ERR_ARG;  // unreachable: at most GBM3D_HOST_NCH chunks
    int launches = 0;
    // the library streams start after whatever the caller queued before this call
    if (cudaEventRecord(g_pipe.start, s) != cudaSuccess ||
        cudaStreamWaitEvent(g_pipe.h2d, g_pipe.start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(g_pipe.comp2, g_pipe.start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(g_pipe.d2h, g_pipe.start, 0) != cudaSuccess)
        return GBM3D_ERR_CUDA;
    // pixels in: per image chunk (B > 1) or, for one image, the pixel rows each chunk of
    // reference rows needs beyond the previous chunk's (its blocks' rows plus the window)
    {
        size_t done_rows = 0;
        for (int c = 0; c < nch; ++c) {
            size_t off, n;
            if (B > 1) {
                off = (size_t)ub[c] * H * W;
                n = (size_t)(ub[c + 1] - ub[c]) * H * W;
            } else {
                const int ylast = std::min((ub[c + 1] - 1) * stride, H - patch);
                const size_t need = (size_t)std::min(H, ylast + patch + radius);
                off = done_rows * W;
                n = need > done_rows ? (need - done_rows) * W : 0;
                done_rows = std::max(done_rows, need);
            }
            if (n && cudaMemcpyAsync(d_img + off, h_imgs + off, n * 2, cudaMemcpyHostToDevice,
                                     g_pipe.h2d) != cudaSuccess)
                return GBM3D_ERR_CUDA;
            if (cudaEventRecord(g_pipe.in[c], g_pipe.h2d) != cudaSuccess) return GBM3D_ERR_CUDA;
        }
    }
    for (int c = 0; c < nch; ++c) {
        const int u0 = ub[c], u1 = ub[c + 1];
        cudaStream_t cs = (c & 1) ? g_pipe.comp2 : s;
        if (cudaStreamWaitEvent(cs, g_pipe.in[c], 0) != cudaSuccess) return GBM3D_ERR_CUDA;
        MatchParams q = p;
        size_t r0, nr;  // first reference and reference count of the chunk in the outputs
        if (B > 1) {
            q.B = u1 - u0;
            q.img = d_img + (size_t)u0 * H * W;
            r0 = (size_t)u0 * per_img_refs;
            nr = (size_t)(u1 - u0) * per_img_refs;
        } else {
            q.img = d_img;
            q.row_begin = u0;
            q.row_end = u1;
            q.out_bstride = (int64_t)(u1 - u0) * p.Rx;
            r0 = (size_t)u0 * p.Rx;
            nr = (size_t)(u1 - u0) * p.Rx;
        }
        q.idx = d_idx + r0 * K;
        q.dist = d_dist + r0 * K;
        q.nvalid = d_nv + r0;
        st = run(q, GBM3D_METHOD_AUTO, cs);
        if (st != GBM3D_OK) return st;
        launches += g_last_launches;
        if (cudaEventRecord(g_pipe.done[c], cs) != cudaSuccess) return GBM3D_ERR_CUDA;
        if (cudaStreamWaitEvent(g_pipe.d2h, g_pipe.done[c], 0) != cudaSuccess) return GBM3D_ERR_CUDA;
        if (cudaMemcpyAsync(h_idx + r0 * K, q.idx, nr * K * 4, cudaMemcpyDeviceToHost, g_pipe.d2h) != cudaSuccess ||
            cudaMemcpyAsync(h_dist + r0 * K, q.dist, nr * K * 4, cudaMemcpyDeviceToHost, g_pipe.d2h) != cudaSuccess)
            return GBM3D_ERR_CUDA;
    }
    // n_valid (small) in one copy after the last chunk
    if (h_n_valid &&
        cudaMemcpyAsync(h_n_valid, d_nv, nref * 4, cudaMemcpyDeviceToHost, g_pipe.d2h) != cudaSuccess)
        return GBM3D_ERR_CUDA;
    g_last_launches = launches;
    // the caller's stream is ordered after the copies out (which follow every chunk's
    // matching), then the call blocks on it
    if (cudaEventRecord(g_pipe.out_done, g_pipe.d2h) != cudaSuccess) return GBM3D_ERR_CUDA;
    if (cudaStreamWaitEvent(s, g_pipe.out_done, 0) != cudaSuccess) return GBM3D_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return GBM3D_ERR_CUDA;
    return GBM3D_OK;
}

int gbm3d_check_range(const int16_t* img, int64_t n, int patch, int* ok, void* stream) {
    if (!img || !ok || n < 1 || patch < 1) return GBM3D_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int* d = nullptr;
    if (cudaMallocAsync((void**)&d, 2 * sizeof(int), s) != cudaSuccess) return GBM3D_ERR_CUDA;
    const int init[2] = {INT_MAX, INT_MIN};
    int h[2];
    cudaError_t e = cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
        range_minmax_kernel<<<blocks, 256, 0, s>>>(img, n, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return GBM3D_ERR_CUDA;
    const long long span = (long long)h[1] - (long long)h[0];
    *ok = ((long long)patch * patch * span * span <= (long long)INT32_MAX) ? 1 : 0;
    return GBM3D_OK;
}

int gbm3d_last_launch_count(void) { return g_last_launches; }

const char* gbm3d_strerror(int status) {
    switch (status) {
        case GBM3D_OK: return "ok";
        case GBM3D_ERR_ARG: return "invalid argument";
        case GBM3D_ERR_RANGE: return "image range violates patch^2*(max-min)^2 <= 2^31-1";
        case GBM3D_ERR_UNSUPPORTED: return "unsupported size (patch > 16, radius > 32, K > 64, or method)";
        case GBM3D_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

#ifndef GBM3D_SRC_ID
#define GBM3D_SRC_ID "unknown"
#endif
// "src <id>": the hash of the sources this library was built from (build.py source_id)
const char* gbm3d_version(void) { return "gbm3d 0.2.0 (sm_100a) src " GBM3D_SRC_ID; }

}  // extern "C"
