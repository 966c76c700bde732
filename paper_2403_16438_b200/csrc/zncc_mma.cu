// ZNCC cross sums on the 5th-generation tensor cores with EXACT integer
// arithmetic: tcgen05.mma kind::i8 (u8 x u8 -> s32 in TMEM), uint16 frames.
//
// For one template patch p the cross sums of all candidates (dy, dx) over a
// tile of 128 frames are one GEMM with the frames as its batch dimension:
//     D[frame m][cand n] = sum_k A[m][k] * B[k][n],  k = bytes of the window,
// A = the raw uint16 window rows as bytes, straight from TMA (a 4-D tensor
// map lands them in the canonical K-major layout [16-byte slice][frame][16 B],
// no conversion pass), so k runs over (pixel, lo/hi byte) pairs;
// B = the template as a fixed-point integer t_u = t_int + 2^23
// (t_int = rint(t_c 2^s), max |t_c| 2^s in [2^21, 2^22)) split into three
// unsigned bytes b0 b1 b2, laid out as four "planes" that pair each frame byte
// with the template byte of the same scale:
//     plane j: B_j[2x] = b_j(x - dx),  B_j[2x + 1] = b_{j-1}(x - dx)   (b_{-1} = b_3 = 0)
// so accumulator j collects sum(lo * b_j + hi * b_{j-1}) and
//     D_total = D0 + 2^8 D1 + 2^16 D2 + 2^24 D3 = sum over the window of f * t_u
// exactly (every partial < 2^31).  The statistics kernel (COMBINE) turns it
// into the covariance with the window sum it forms anyway:
//     X = D_total - 2^23 sum f,   cov = (X - sum f * T / n) 2^-s,  T = sum t_int,
// then z = cov * inv and the group partials in float64.  Products and sums
// are exact; the only approximation is the template's fixed-point rounding
// (2^-22 of the patch's largest deviation from its mean).
//
// Work: one CTA (4 warps) per (patch, 128-frame tile); candidates in passes of
// up to 128 columns (4 accumulators x 128 = all 512 TMEM columns); the window
// row by row through a two-stage ring: thread 0 issues the row's A box by TMA,
// all threads expand the four B planes from pre-shifted template rows (one
// aligned 16-byte load per 16-byte vector), then thread 0 issues
// 4 x (2 WXP / 32) MMAs (M = 128, N <= 128, K = 32) and commits to the
// stage's "empty" barrier; the next row's staging overlaps them.  The
// epilogue (tcgen05.ld) combines the four accumulators into int64 D_total.
#include "tma.cuh"
#include "vb.cuh"

#include <cudaTypedefs.h>

namespace vb {

namespace {

constexpr int kM = 128;          // frames per tile (UMMA M)
constexpr int kBThreads = 256;   // B-producer threads (warps 6-13)
constexpr int kThreads = 6 * 32 + kBThreads;
constexpr int kNMax = 128;       // candidates per pass (per accumulator)
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxStages = 6;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // SWIZZLE_NONE, K-major
}
// K-major, 128-byte swizzle (SBO = 1024: 8 rows of 128 B per swizzle atom)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::i8: D s32 (bits 4-5 = 2), A u8 (bits 7-9 = 0), B s8 (bits 10-12 = 1), K-major A and B
__host__ __device__ constexpr uint32_t idesc_u8s8(int M, int N) {
    return (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
}  // namespace

struct MmaArgs {
    int64_t n_frames;
    int tma_z0;
    int P, R, S, SS;
    int rows;              // window rows P + 2R
    int tpw, toff;         // pre-shifted digit row width and tx offset
    int npass, na, nb;     // passes; A ring and B ring depths
    int np[8];             // candidates per pass (multiples of 16, <= 128)
    int off_b, b_bytes, off_tq;  // B ring offset, bytes per B slot, staged digit planes
    const int32_t* origins;
    const int8_t* tq;      // [N][3 digit planes][8 shifts][P][tpw]
    const double* tscale;  // [N] 2^-s
    float* cov;            // [n_frames][N][ss_pad] covariance of each window with the template patch
    int ss_pad;
};

// Template prep for the tensor-core path (once per reference), one CTA per
// patch: the fixed-point exponent s (max |t_c| 2^s in [2^21, 2^22)),
// t_int = rint(t_c 2^s) adjusted so that sum t_int = 0 exactly (the
// |T| <= n/2 elements rounded furthest the wrong way move by one unit), so
// sum f * t_int is the covariance of the window with the quantised template
// for any window -- no sum-of-f correction -- and t_int in balanced base-256
// digits d0 + 2^8 d1 + 2^16 d2 (each in [-128, 127], signed bytes), stored as
// zero-padded rows x = tx + toff in eight copies shifted by 0..7 pixels (copy
// q holds row[x + q]), so every 8-pixel slice of a digit plane is one aligned
// 8-byte load.
__global__ void mma_prep_kernel(const float* __restrict__ tmpl, int P, int tp, int tpw, int toff,
                                int8_t* __restrict__ tq, double* __restrict__ tscale) {
    const int p = blockIdx.x;
    const float* t = tmpl + (size_t)p * P * tp;
    extern __shared__ int s_ti[];  // [P*P] t_int
    __shared__ float s_max[32];
    __shared__ int s_s;
    float mx = 0.0f;
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) mx = fmaxf(mx, fabsf(t[(i / P) * tp + i % P]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f;
        for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) m = fmaxf(m, s_max[i]);
        int ex = 0;
        if (m > 0.0f) frexpf(m, &ex);  // m = f 2^ex, f in [0.5, 1): m 2^(22 - ex) in [2^21, 2^22)
        s_s = m > 0.0f ? 22 - ex : 0;
        tscale[p] = ldexp(1.0, -s_s);
    }
    __syncthreads();
    const int sc = s_s;
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) s_ti[i] = (int)rint(ldexp((double)t[(i / P) * tp + i % P], sc));
    __syncthreads();
    if (threadIdx.x == 0) {  // sum t_int = 0: move the elements rounded furthest the wrong way
        long long tot = 0;
        for (int i = 0; i < P * P; ++i) tot += s_ti[i];
        while (tot != 0) {
            const int dir = tot > 0 ? -1 : 1;
            int best = -1;
            double bres = 0.0;
            for (int i = 0; i < P * P; ++i) {
                const double res = (ldexp((double)t[(i / P) * tp + i % P], sc) - (double)s_ti[i]) * (double)dir;
                if (best < 0 || res > bres) {
                    best = i;
                    bres = res;
                }
            }
            s_ti[best] += dir;
            tot += dir;
        }
    }
    __syncthreads();
    int8_t* out = tq + (size_t)p * 3 * 8 * P * tpw;
    for (int i = threadIdx.x; i < 8 * P * tpw; i += blockDim.x) {
        const int q = i / (P * tpw), rem = i - q * P * tpw, ty = rem / tpw, x = rem - ty * tpw;
        const int tx = x + q - toff;
        int v = (tx >= 0 && tx < P) ? s_ti[ty * P + tx] : 0;
        for (int j = 0; j < 3; ++j) {  // balanced base-256 digits
            const int d = ((v + 128) & 255) - 128;
            out[((size_t)(j * 8 + q) * P) * tpw + rem] = (int8_t)d;
            v = (v - d) / 256;
        }
    }
}

// Warp roles: warp 0 lane 0 issues the A rows by TMA; warp 1 lane 0 issues
// the MMAs (and owns TMEM); warps 2-5 are the epilogue (TMEM lane quadrants
// 2, 3, 0, 1 -> frames); warps 6-13 expand the B planes.  Stage ring of
// nstages (A row + B planes): fullA (TMA bytes), fullB (256 producer
// arrivals), empty (MMA commit); per pass tmem_full (last commit) and
// tmem_empty (128 epilogue arrivals) hand the accumulators over.
__global__ void __launch_bounds__(kThreads, 1) zncc_mma_kernel(MmaArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t fullA[kMaxStages], emptyA[kMaxStages], fullB[kMaxStages], emptyB[kMaxStages];
    __shared__ __align__(8) uint64_t tmem_full, tmem_empty;
    const int p = blockIdx.x;
    const int64_t t0 = (int64_t)blockIdx.y * kM;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = a.P, S = a.S, rows = a.rows, na = a.na, nb = a.nb;
    const int px = a.origins[2 * p], py = a.origins[2 * p + 1];
    const int x0 = px - a.R, y0 = py - a.R;
    const int xa = x0 & ~7, o = x0 - xa;  // A rows start 16-byte aligned; B absorbs the offset
    const int8_t* tqg = a.tq + (size_t)p * 3 * 8 * P * a.tpw;
    int8_t* tqs = reinterpret_cast<int8_t*>(sm + a.off_tq);  // the patch's digit planes, staged once
    const int tq_vec = (3 * 8 * P * a.tpw + 15) / 16;
    const int n_it = a.npass * rows;

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int b = 0; b < na; ++b) {
            mbar_init(&fullA[b], 1);
            mbar_init(&emptyA[b], 1);
        }
        for (int b = 0; b < nb; ++b) {
            mbar_init(&fullB[b], kBThreads);
            mbar_init(&emptyB[b], 1);
        }
        mbar_init(&tmem_full, 1);
        mbar_init(&tmem_empty, 128);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    for (int v = tid; v < tq_vec; v += kThreads)
        reinterpret_cast<uint4*>(tqs)[v] = __ldg(reinterpret_cast<const uint4*>(tqg) + v);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        // ---- A producer ----
        if (lane == 0) {
            for (int it = 0; it < n_it; ++it) {
                const int st = it % na;
                if (it >= na) mbar_wait(&emptyA[st], (uint32_t)(((it / na) - 1) & 1));
                mbar_expect_tx(&fullA[st], (uint32_t)(kM * 128));
                tma_load_3d(sm + (size_t)st * kM * 128, &tmap, xa, y0 + it % rows, a.tma_z0 + (int)t0, &fullA[st]);
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer ----
        if (lane == 0) {
            int it = 0, base = 0;
            for (int pass = 0; pass < a.npass; ++pass) {
                const int np = a.np[pass];
                const uint32_t idesc = idesc_u8s8(kM, np);
                if (pass > 0) mbar_wait(&tmem_empty, (uint32_t)((pass - 1) & 1));  // accumulators read out
                for (int r = 0; r < rows; ++r, ++it) {
                    const int sa = it % na, sb = it % nb;
                    mbar_wait(&fullA[sa], (uint32_t)((it / na) & 1));
                    mbar_wait(&fullB[sb], (uint32_t)((it / nb) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    const uint32_t a0 = smem_u32(sm + (size_t)sa * kM * 128);
                    const uint32_t b0 = smem_u32(sm + a.off_b + (size_t)sb * a.b_bytes);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int s = 0; s < 4; ++s)  // K = 128 bytes = 4 x K32 inside the swizzle atom
                            umma_i8(tmem + j * kNMax, sdesc_sw128(a0 + 32 * s), sdesc_sw128(b0 + j * np * 128 + 32 * s),
                                    idesc, (r > 0 || s > 0) ? 1u : 0u);
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&emptyA[sa])));
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&emptyB[sb])));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&tmem_full)));
                base += np;
            }
        }
    } else if (warp < 6) {
        // ---- epilogue: TMEM lane quadrant warp % 4 -> frames ----
        const int quad = warp & 3;
        const int m = quad * 32 + lane;
        const int64_t t = t0 + m;
        const double scale = a.tscale[p];
        int base = 0;
        for (int pass = 0; pass < a.npass; ++pass) {
            const int np = a.np[pass];
            mbar_wait(&tmem_full, (uint32_t)(pass & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            float* out = a.cov + ((size_t)t * gridDim.x + p) * a.ss_pad + base;
            const int ncols = min(np, a.SS - base);
            for (int c0 = 0; c0 < np; c0 += 16) {
                uint32_t v[4][16];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                        : "=r"(v[j][0]), "=r"(v[j][1]), "=r"(v[j][2]), "=r"(v[j][3]), "=r"(v[j][4]), "=r"(v[j][5]),
                          "=r"(v[j][6]), "=r"(v[j][7]), "=r"(v[j][8]), "=r"(v[j][9]), "=r"(v[j][10]), "=r"(v[j][11]),
                          "=r"(v[j][12]), "=r"(v[j][13]), "=r"(v[j][14]), "=r"(v[j][15])
                        : "r"(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(j * kNMax + c0)));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n");
                if (t < a.n_frames) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (c0 + i < ncols) {
                            const long long x = (long long)(int)v[0][i] + ((long long)(int)v[1][i] << 8) +
                                                ((long long)(int)v[2][i] << 16) + ((long long)(int)v[3][i] << 24);
                            out[c0 + i] = (float)((double)x * scale);  // the exact covariance, rounded once
                        }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            mbar_arrive_cta(&tmem_empty);
            base += np;
        }
    } else {
        // ---- B producers: thread -> (candidate n, half of the 8 chunks) ----
        const int bt = tid - 6 * 32;
        const int n = bt & (kNMax - 1), c_lo = (bt >> 7) * 4;
        int it = 0, base = 0;
        for (int pass = 0; pass < a.npass; ++pass) {
            const int np = a.np[pass];
            const int g = base + n;
            const bool cand = n < np && g < a.SS;
            const int dy = cand ? g / S : -1, dx = cand ? g % S : 0;
            const int xs0 = -o - dx + a.toff;  // chunk c starts at pixel 8 c + xs0 of the padded row
            const int q = xs0 & 7;             // pre-shifted copy that makes every slice 8-byte aligned
            for (int r = 0; r < rows; ++r, ++it) {
                const int st = it % nb;
                if (it >= nb) mbar_wait(&emptyB[st], (uint32_t)(((it / nb) - 1) & 1));  // slot free
                if (n < np) {  // plane j = (d_j, d_{j-1}) byte pairs, 128-byte swizzled rows
                    unsigned char* drow = sm + a.off_b + (size_t)st * a.b_bytes + (size_t)n * 128;
                    const int ty = r - dy;
                    const bool live = cand && ty >= 0 && ty < P;
                    const int8_t* row = tqs + ((size_t)q * P + (live ? ty : 0)) * a.tpw + (xs0 - q);
                    const size_t pstride = (size_t)8 * P * a.tpw;
#pragma unroll
                    for (int c = c_lo; c < c_lo + 4; ++c) {
                        uint2 d0 = make_uint2(0u, 0u), d1 = d0, d2 = d0;
                        if (live) {
                            d0 = *reinterpret_cast<const uint2*>(row + 8 * c);
                            d1 = *reinterpret_cast<const uint2*>(row + pstride + 8 * c);
                            d2 = *reinterpret_cast<const uint2*>(row + 2 * pstride + 8 * c);
                        }
                        const uint2 dj[5] = {make_uint2(0u, 0u), d0, d1, d2, make_uint2(0u, 0u)};
                        const int sw = ((c ^ (n & 7)) << 4);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {  // (lo-byte weight, hi-byte weight) = (d_j, d_{j-1})
                            const uint2 lo = dj[j + 1], hi = dj[j];
                            const uint4 v = make_uint4(__byte_perm(lo.x, hi.x, 0x5140), __byte_perm(lo.x, hi.x, 0x7362),
                                                       __byte_perm(lo.y, hi.y, 0x5140), __byte_perm(lo.y, hi.y, 0x7362));
                            *reinterpret_cast<uint4*>(drow + (size_t)j * np * 128 + sw) = v;
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_arrive_cta(&fullB[st]);
            }
            base += np;
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
}

// ---------------------------------------------------------------- host side
bool mma_supported(int patch, int radius, int dtype) {
    const int S = 2 * radius + 1;
    return dtype == VB_U16 && patch >= 1 && patch <= 32 && patch + S - 1 + 7 <= 64 && knob("VB_ZNCC_MMA", 0) != 0 &&
           mma_geom(patch, radius).smem <= 227 * 1024;
}

MmaGeom mma_geom(int patch, int radius) {
    MmaGeom g;
    const int S = 2 * radius + 1, SS = S * S;
    g.wx = patch + 2 * radius;
    g.wxp = 64;                           // one 128-byte swizzled row of 64 pixels per frame
    g.toff = S - 1 + 7;                   // every chunk start 8 c - o - dx + toff >= 0
    g.tpw = (g.toff + g.wxp + 7) / 8 * 8;
    g.nchunks = g.wx;                     // one window row per stage
    const size_t tq = (size_t)3 * 8 * patch * g.tpw;
    const size_t a_bytes = (size_t)kM * 128;
    // A ring (one 16 KB row per slot) deep enough to hide the TMA latency, B ring
    // double-buffered, widest pass (per accumulator) that fits beside them
    const int na = knob("VB_MMA_ASTAGES", 4), nb = knob("VB_MMA_BSTAGES", 2);
    int nmax = kNMax;
    auto b_of = [&](int nm) { return 4 * (size_t)nm * 128; };
    while (nmax > 16 && na * a_bytes + nb * b_of(nmax) + tq > 227 * 1024 - 2048) nmax -= 16;
    g.na = na;
    g.nb = nb;
    g.npass = (SS + nmax - 1) / nmax;
    int left = SS;
    for (int i = 0; i < 8; ++i) {
        const int n = std::min(nmax, std::max(0, left));
        g.np[i] = (n + 15) / 16 * 16;
        left -= n;
    }
    g.off_a = 0;
    g.off_b = na * a_bytes;
    g.b_bytes = b_of(nmax);
    g.off_tq = g.off_b + nb * g.b_bytes;
    g.smem = g.off_tq + tq;
    if (g.npass > 8) g.smem = (size_t)1 << 30;  // unsupported
    return g;
}

int launch_mma_prep(const Templates& t, int patch, int radius, cudaStream_t s) {
    const MmaGeom g = mma_geom(patch, radius);
    mma_prep_kernel<<<t.n, 128, patch * patch * sizeof(int), s>>>(t.tmpl, patch, t.tp, g.tpw, g.toff,
                                                                  static_cast<int8_t*>(t.t16), t.tscale);
    VB_LAUNCHED();
    return VB_OK;
}

// frames [T][H][W] uint16 as {W, H, T} with a box of {64 pixels, 1 row, 128
// frames} and 128-byte swizzle: one window row of 128 frames lands as the
// K-major SWIZZLE_128B A tile ([frame][128 B], 8-frame atoms of 1,024 B).
bool make_frames_tmap_sw128(CUtensorMap* map, const void* base, int64_t t, int h, int w) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
    }
    if (!encode || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (w & 7)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)(t > 0 ? t : 1)};
    cuuint64_t strides[2] = {(cuuint64_t)w * 2, (cuuint64_t)h * w * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kM};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int launch_zncc_mma(const Templates& t, int patch, int radius, int64_t n_frames, int tma_z0, const CUtensorMap& tmap,
                    float* cov, int ss_pad, cudaStream_t s) {
    if (n_frames <= 0) return VB_OK;
    const MmaGeom g = mma_geom(patch, radius);
    if (g.npass > 8 || g.smem > 227 * 1024) return fail(VB_EINVAL, "search window too large for the tensor-core path");
    MmaArgs a;
    a.n_frames = n_frames;
    a.tma_z0 = tma_z0;
    a.P = patch;
    a.R = radius;
    a.S = 2 * radius + 1;
    a.SS = a.S * a.S;
    a.rows = g.wx;
    a.tpw = g.tpw;
    a.toff = g.toff;
    a.npass = g.npass;
    a.na = g.na;
    a.nb = g.nb;
    for (int i = 0; i < 8; ++i) a.np[i] = g.np[i];
    a.off_b = (int)g.off_b;
    a.b_bytes = (int)g.b_bytes;
    a.off_tq = (int)g.off_tq;
    a.origins = t.origins;
    a.tq = static_cast<const int8_t*>(t.t16);
    a.tscale = t.tscale;
    a.cov = cov;
    a.ss_pad = ss_pad;
    VB_CUDA(cudaFuncSetAttribute(zncc_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    for (int64_t f0 = 0; f0 < n_frames; f0 += (int64_t)65535 * kM) {
        const int64_t nf = std::min<int64_t>((int64_t)65535 * kM, n_frames - f0);
        MmaArgs b = a;
        b.n_frames = nf;
        b.tma_z0 = tma_z0 + (int)f0;
        b.cov = cov + (size_t)f0 * t.n * ss_pad;
        dim3 grid((unsigned)t.n, (unsigned)((nf + kM - 1) / kM));
        {
            ProfScope ps(kProfZncc, s);
            zncc_mma_kernel<<<grid, kThreads, g.smem, s>>>(b, tmap);
        }
        VB_LAUNCHED();
    }
    return VB_OK;
}

}  // namespace vb
