// ZNCC cross sums on the 5th-generation tensor cores (tcgen05.mma kind::f16,
// f32 accumulation in TMEM) for uint16 camera frames -- the go/no-go
// PROTOTYPE of VERDICT r01 item 7, compiled but reachable only in the
// experiment build (VB_ZNCC_MMA=1).  Measured on C2 (scripts/mma_check.py,
// profiles/r02_mma_prototype.json): correct integer shifts, but score error
// 3.8e-7 vs the float64 oracle (FFMA path 4.1e-8; C1 1.04e-6 > the 1e-6
// bound: the tensor core's f32 accumulation over 190 K-steps is not
// round-to-nearest) and 3.4 ms of MMA kernel per 1,000 C2 frames against
// 1.45 ms for the FFMA search -- no-go; see DESIGN.md for the exact int8
// variant and its estimated ceiling.
//
// For one template patch p the cross sums of all candidates (dy, dx) over a
// tile of 128 frames are one GEMM
//     D[frame m][cand n] = sum_k A[m][k] * B[k][n],
// k = window pixel (wy, wx) of the (P + 2R)^2 search window,
// A[m][k] = frame_m(window pixel k) - c   (integer, c = the group's centre),
// B[k][n] = t_c[wy - dy][wx - dx]          (0 outside the patch),
// i.e. the template patch expanded into its Toeplitz (correlation) matrix,
// shared by every frame -- the frames are the GEMM's batch dimension.
//
// Exactness: A is split as v = 2048 q + m with m in [-1024, 1024) and q in
// [-32, 32], both exact in f16; the centred template t_c (f32) is scaled by
// a power of two into [8, 16) and split into t_hi = f16(t_s) and
// t_lo = f16(t_s - t_hi).  Products are exact in the f32 accumulator; the
// q sweep (frames with samples more than 1024 counts from the centre) runs
// only when a tile needs it and adds exact zeros otherwise, so a frame's
// result never depends on the other frames of its tile.  D * 2^-e is the
// cross sum the FFMA kernels form (zncc_group_kernel), accumulated in a
// different order.
//
// Work: one CTA per (patch, 128-frame tile); candidates in passes of NP
// columns (TMEM accumulator [128 lanes][NP] f32); the window in chunks of two
// rows: per chunk the two raw rows of all 128 frames land by TMA (one box
// {56 cols, 1 row, 128 frames} per row), all threads convert them into the
// K-major A tile and expand the template rows into the K-major B tiles
// (t_hi, t_lo), one elected thread issues 2 x (2 WXP / 16) MMAs (M = 128,
// N = NP, K = 16) and commits to an mbarrier.  Two CTAs per SM overlap one's
// staging with the other's MMAs.  The epilogue writes cov[t][p][n] (f32);
// zncc_stats_kernel<..., COMBINE> then forms z = cov * inv per patch and the
// group partials.
#include <cuda_fp16.h>

#include "tma.cuh"
#include "vb.cuh"

namespace vb {

namespace {

constexpr int kM = 128;          // frames per tile (UMMA M)
constexpr int kThreads = 128;
constexpr int kRawW = 56;        // raw TMA box width (u16): 112 B rows, conflict-free 16 B reads
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // SWIZZLE_NONE, K-major
}
// kind::f16: D f32 (bit 4), A f16 (bits 7-9 = 0), B f16 (bits 10-12 = 0), K-major A and B
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tma_load_3d_box(void* dst, const CUtensorMap* map, int x, int y, int z,
                                                uint64_t* bar) {
    tma_load_3d(dst, map, x, y, z, bar);
}

// Two raw rows of all kM frames -> the K-major A tile: thread (row r, frame m)
// reads its row as aligned 16-byte words (conflict-free: 112-byte rows), takes
// the 8-sample groups starting at the window's column offset O (compile-time
// funnel), centres them exactly (v = u16 - c as an f32 integer) and writes
// m = v - 2048 q (first sweep) or q (second sweep) as f16, q = floor((v + 1024) / 2048).
template <int O>
__device__ __forceinline__ void convert_rows(const uint16_t* raw, unsigned char* sA, int gpr, uint32_t sbo,
                                             float magic, int sweep, int& qflag, int tid) {
    for (int u = tid; u < 2 * kM; u += kThreads) {
        const int r = u / kM, m = u - r * kM;
        const uint4* src = reinterpret_cast<const uint4*>(raw + ((size_t)r * kM + m) * kRawW);
        unsigned char* dst = sA + (m >> 3) * sbo + (m & 7) * 16 + r * gpr * 128;
        uint4 cur = src[0];
#pragma unroll 1
        for (int g = 0; g < gpr; ++g) {
            const uint4 nxt = src[g + 1];
            const uint32_t w[8] = {cur.x, cur.y, cur.z, cur.w, nxt.x, nxt.y, nxt.z, nxt.w};
            uint32_t hv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t pair = (O % 2 == 0) ? w[O / 2 + i] : __byte_perm(w[O / 2 + i], w[O / 2 + i + 1], 0x5432);
                const float v0 = __fsub_rn(__uint_as_float(0x4B000000u | (pair & 0xFFFFu)), magic);
                const float v1 = __fsub_rn(__uint_as_float(0x4B000000u | (pair >> 16)), magic);
                const float q0 = floorf(__fmul_rn(__fadd_rn(v0, 1024.0f), 1.0f / 2048.0f));
                const float q1 = floorf(__fmul_rn(__fadd_rn(v1, 1024.0f), 1.0f / 2048.0f));
                qflag |= (q0 != 0.0f) | (q1 != 0.0f);
                const float e0 = sweep ? q0 : __fsub_rn(v0, __fmul_rn(2048.0f, q0));
                const float e1 = sweep ? q1 : __fsub_rn(v1, __fmul_rn(2048.0f, q1));
                const __half2 h = __floats2half2_rn(e0, e1);
                hv[i] = *reinterpret_cast<const uint32_t*>(&h);
            }
            *reinterpret_cast<uint4*>(dst + g * 128) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
            cur = nxt;
        }
    }
}

}  // namespace

struct MmaArgs {
    int64_t n_frames;
    int tma_z0;
    int P, R, S, SS, ss_pad;
    int wx, wxp, nchunks;  // window width, padded to 8; two-row chunks
    int np, npass;         // candidates per pass (multiple of 16), passes
    int tpw, toff;         // t16 row width and tx offset
    int off_a, off_b;      // shared-memory carve-up (raw boxes at 0)
    const int32_t* origins;
    const int32_t* cen;
    const __half* t16;     // [N][8 shifts][2 parts][P][tpw]
    const float* tscale;   // [N] 2^-e
    float* cov;            // [n_frames][N][ss_pad]
};

// Template prep for the tensor-core path (once per reference): per patch the
// exponent e with max|t_c| 2^e in [8, 16), the f16 split t_hi / t_lo of
// t_s = t_c 2^e stored as zero-padded rows x = tx + toff in eight copies
// shifted by s = 0..7 elements (copy s holds row[x + s]), so every 8-wide
// slice the B expansion needs is one aligned 16-byte load; and the centre c
// of the patch's group (the FFMA kernels' group_centre).
__global__ void mma_prep_kernel(const float* __restrict__ tmpl, int P, int tp, int tpw, int toff,
                                const double* __restrict__ rmean, const PatchGroup* __restrict__ groups,
                                const int32_t* __restrict__ patch_group, __half* __restrict__ t16,
                                float* __restrict__ tscale, int32_t* __restrict__ cen) {
    const int p = blockIdx.x;
    const float* t = tmpl + (size_t)p * P * tp;
    __shared__ float s_max[32];
    __shared__ int s_e;
    float mx = 0.0f;
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) mx = fmaxf(mx, fabsf(t[(i / P) * tp + i % P]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f;
        for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) m = fmaxf(m, s_max[i]);
        int ex = 0;
        if (m > 0.0f) frexpf(m, &ex);  // m = f 2^ex, f in [0.5, 1)
        const int e = m > 0.0f ? 4 - ex : 0;
        s_e = e;
        tscale[p] = ldexpf(1.0f, -e);
        const PatchGroup g = groups[patch_group[p]];
        double mm = 0.0;
        for (int q = 0; q < g.count; ++q) mm += rmean[g.first + q];
        mm /= (double)g.count;
        cen[p] = fabs(mm) >= 64.0 ? (int32_t)rint(mm) : 0;  // group_centre (motion.cu)
    }
    __syncthreads();
    const int e = s_e;
    __half* out = t16 + (size_t)p * 8 * 2 * P * tpw;
    for (int i = threadIdx.x; i < 8 * P * tpw; i += blockDim.x) {
        const int s = i / (P * tpw), rem = i - s * P * tpw, ty = rem / tpw, x = rem - ty * tpw;
        const int tx = x + s - toff;
        float ts = 0.0f;
        if (tx >= 0 && tx < P) ts = ldexpf(t[ty * tp + tx], e);
        const __half hi = __float2half_rn(ts);
        const __half lo = __float2half_rn(ts - __half2float(hi));
        out[((size_t)s * 2 + 0) * P * tpw + rem] = hi;
        out[((size_t)s * 2 + 1) * P * tpw + rem] = lo;
    }
}

__global__ void __launch_bounds__(kThreads, 2) zncc_mma_kernel(MmaArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar_raw, bar_mma;
    __shared__ int16_t s_nmap[2 * 256];  // pass candidate n -> (dy, dx), -1 = padding
    const int p = blockIdx.x;
    const int64_t t0 = (int64_t)blockIdx.y * kM;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = a.P, R = a.R, S = a.S, wxp = a.wxp, np = a.np;
    const int gpr = wxp / 8;        // K groups (8 pixels) per window row
    const int kgroups = 2 * gpr;    // per chunk
    const int ksteps = kgroups / 2; // K16 steps per chunk
    const int px = a.origins[2 * p], py = a.origins[2 * p + 1];
    const int x0 = px - R, y0 = py - R;
    const int xa = x0 & ~7, o = x0 - xa;
    const int cen = a.cen[p];
    const float magic = 8388608.0f + (float)cen;
    const __half* tp16 = a.t16 + (size_t)p * 8 * 2 * P * a.tpw;
    uint16_t* raw = reinterpret_cast<uint16_t*>(sm);
    unsigned char* sA = sm + a.off_a;
    unsigned char* sB = sm + a.off_b;
    const uint32_t sbo = (uint32_t)kgroups * 128;  // 8-row core-matrix groups (A: frames, B: candidates)
    const uint32_t b_part = (uint32_t)np * kgroups * 16;  // bytes of one B part

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(&bar_raw, 1);
        mbar_init(&bar_mma, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    uint32_t ph_raw = 0, ph_mma = 0;
    bool mma_pending = false;
    auto fetch_raw = [&](int c) {  // window rows 2c, 2c+1 of frames t0.. (zero-filled out of bounds)
        if (tid == 0) {
            mbar_expect_tx(&bar_raw, (uint32_t)(2 * kM * kRawW * 2));
            for (int r = 0; r < 2; ++r)
                tma_load_3d_box(raw + (size_t)r * kM * kRawW, &tmap, xa, y0 + 2 * c + r, a.tma_z0 + (int)t0, &bar_raw);
        }
    };
    const uint32_t idesc = idesc_f16(kM, np);
    int qflag_any = 0;
#pragma unroll 1
    for (int pass = 0; pass < a.npass; ++pass) {
        // candidate map of this pass
        for (int n = tid; n < np; n += kThreads) {
            const int g = pass * np + n;
            s_nmap[2 * n] = g < a.SS ? (int16_t)(g / S) : (int16_t)-1;
            s_nmap[2 * n + 1] = g < a.SS ? (int16_t)(g % S) : (int16_t)0;
        }
#pragma unroll 1
        for (int sweep = 0; sweep < 2; ++sweep) {
            if (sweep == 1 && !qflag_any) break;  // no sample of the tile is >= 1024 from the centre
            fetch_raw(0);
            int qflag = 0;
#pragma unroll 1
            for (int c = 0; c < a.nchunks; ++c) {
                mbar_wait(&bar_raw, ph_raw);
                ph_raw ^= 1u;
                if (mma_pending) {  // the previous chunk's MMAs have read A and B
                    mbar_wait(&bar_mma, ph_mma);
                    ph_mma ^= 1u;
                    mma_pending = false;
                }
                // ---- A: raw rows -> K-major f16 (m part or q part) ----
                switch (o) {
                    case 0: convert_rows<0>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 1: convert_rows<1>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 2: convert_rows<2>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 3: convert_rows<3>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 4: convert_rows<4>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 5: convert_rows<5>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    case 6: convert_rows<6>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                    default: convert_rows<7>(raw, sA, gpr, sbo, magic, sweep, qflag, tid); break;
                }
                // ---- B: Toeplitz expansion of template rows (t_hi, t_lo; x 2048 in the q sweep) ----
                const int nvec = np * kgroups;
                for (int v = tid; v < 2 * nvec; v += kThreads) {
                    const int part = v >= nvec ? 1 : 0;
                    const int vv = v - part * nvec;
                    const int gk = vv / np, n = vv - gk * np;
                    const int r = gk >= gpr ? 1 : 0, g = gk - r * gpr;
                    const int dy = s_nmap[2 * n], dx = s_nmap[2 * n + 1];
                    const int ty = 2 * c + r - dy;
                    uint4 val = make_uint4(0u, 0u, 0u, 0u);
                    if (dy >= 0 && ty >= 0 && ty < P) {
                        const int xs = 8 * g - dx + a.toff;  // first element of the slice in the padded row
                        const int s = xs & 7;
                        val = __ldg(reinterpret_cast<const uint4*>(tp16 + (((size_t)s * 2 + part) * P + ty) * a.tpw +
                                                                   (xs - s)));
                        if (sweep) {
                            __half2* hp = reinterpret_cast<__half2*>(&val);
                            const __half2 k2048 = __floats2half2_rn(2048.0f, 2048.0f);
#pragma unroll
                            for (int j = 0; j < 4; ++j) hp[j] = __hmul2(hp[j], k2048);
                        }
                    }
                    *reinterpret_cast<uint4*>(sB + part * b_part + (n >> 3) * sbo + (n & 7) * 16 + gk * 128) = val;
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncthreads();
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                if (c + 1 < a.nchunks) fetch_raw(c + 1);  // the raw rows are converted
                if (tid == 0) {
                    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
#pragma unroll 1
                    for (int part = 0; part < 2; ++part)
#pragma unroll 1
                        for (int s = 0; s < ksteps; ++s) {
                            const uint64_t da = sdesc(a0 + s * 256, 128, sbo);
                            const uint64_t db = sdesc(b0 + part * b_part + s * 256, 128, sbo);
                            const uint32_t acc = (sweep > 0 || c > 0 || part > 0 || s > 0) ? 1u : 0u;
                            umma_f16(tmem, da, db, idesc, acc);
                        }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&bar_mma)));
                }
                mma_pending = true;
            }
            if (sweep == 0) qflag_any = __syncthreads_or(qflag);
        }
        // ---- epilogue: D (TMEM lane = frame) -> cov rows ----
        mbar_wait(&bar_mma, ph_mma);
        ph_mma ^= 1u;
        mma_pending = false;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int m = warp * 32 + lane;
        const int64_t t = t0 + m;
        const float sc = a.tscale[p];
        float* out = a.cov + ((size_t)t * gridDim.x + p) * a.ss_pad + pass * np;
        const int ncols = min(np, a.SS - pass * np);
#pragma unroll 1
        for (int c0 = 0; c0 < np; c0 += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            if (t < a.n_frames) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < ncols) out[c0 + j] = __fmul_rn(__uint_as_float(v[j]), sc);
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();  // TMEM read before the next pass overwrites it
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
}

// ---------------------------------------------------------------- host side
bool mma_supported(int patch, int radius, int dtype) {
    const int S = 2 * radius + 1;
    // measured no-go (profiles/r02_mma_prototype.json): experiment build only
    return dtype == VB_U16 && patch >= 1 && patch <= 32 && S <= 25 && knob("VB_ZNCC_MMA", 0) != 0;
}

MmaGeom mma_geom(int patch, int radius) {
    MmaGeom g;
    const int S = 2 * radius + 1, SS = S * S;
    g.wx = patch + 2 * radius;
    g.wxp = (g.wx + 7) / 8 * 8;
    g.toff = (S - 1 + 7) / 8 * 8;
    g.tpw = (g.toff + g.wxp + 7) / 8 * 8;
    g.npass = (SS + 223) / 224;
    g.np = ((SS + g.npass - 1) / g.npass + 15) / 16 * 16;
    g.nchunks = (g.wx + 1) / 2;
    const int kgroups = 2 * g.wxp / 8;
    g.off_a = ((2 * kM * kRawW * 2) + 127) / 128 * 128;
    g.off_b = g.off_a + kM * kgroups * 16;
    g.smem = g.off_b + 2 * g.np * kgroups * 16;
    return g;
}

int launch_mma_prep(const Templates& t, int patch, int radius, cudaStream_t s) {
    const MmaGeom g = mma_geom(patch, radius);
    mma_prep_kernel<<<t.n, 128, 0, s>>>(t.tmpl, patch, t.tp, g.tpw, g.toff, t.rmean, t.groups, t.patch_group, static_cast<__half*>(t.t16),
                                        t.tscale, t.cen);
    VB_LAUNCHED();
    return VB_OK;
}

int launch_zncc_mma(const Templates& t, int h, int w, int patch, int radius, const void* frames, int64_t n_frames,
                    int tma_z0, const CUtensorMap& tmap, float* cov, int ss_pad, cudaStream_t s) {
    (void)h;
    (void)w;
    (void)frames;
    if (n_frames <= 0) return VB_OK;
    const MmaGeom g = mma_geom(patch, radius);
    MmaArgs a;
    a.n_frames = n_frames;
    a.tma_z0 = tma_z0;
    a.P = patch;
    a.R = radius;
    a.S = 2 * radius + 1;
    a.SS = a.S * a.S;
    a.ss_pad = ss_pad;
    a.wx = g.wx;
    a.wxp = g.wxp;
    a.nchunks = g.nchunks;
    a.np = g.np;
    a.npass = g.npass;
    a.tpw = g.tpw;
    a.toff = g.toff;
    a.off_a = g.off_a;
    a.off_b = g.off_b;
    a.origins = t.origins;
    a.cen = t.cen;
    a.t16 = static_cast<const __half*>(t.t16);
    a.tscale = t.tscale;
    a.cov = cov;
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
