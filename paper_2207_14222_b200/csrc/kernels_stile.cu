// kernels_stile.cu -- strided-axis FFT passes with a TMA-prefetched tile
// (the default y/z passes for line lengths 64..1024 on sm_100a).
//
// A CTA owns COLS = 16 adjacent columns (128-byte rows) x N rows of a strided
// axis (y: stride nx; z: stride nx*ny) per tile and walks its tiles in a
// persistent loop.  One thread issues the tensor-map TMA boxes
// (cp.async.bulk.tensor, SASS UTMALDG) of tile i+1 into the single stage as
// soon as every thread has copied tile i into registers, so the load of the
// next tile overlaps the whole FFT arithmetic of the current one; results are
// stored straight from registers (128-byte rows).  Thread (c, j) owns column
// c, rows j + N1*m (the four-step layout of fft_core.cuh).
//
// Shared memory per CTA: stage (COLS*N float2) + exchange buffer + twiddles.
// For N = 1024 the exchange buffer is HALF a tile (64 KB), so stage +
// exchange fit one SM (200 KB): the transpose of the four-step FFT runs in
// two rounds.  Round r moves, for every writer row n1, the half of its k2
// values with k2 >> (L2-1) == r ^ b(n1), b(n1) = top bit of n1; to keep the
// register indices compile-time, the half a thread writes/reads first is
// selected by DFT shift identities instead of register swaps:
//   x'[n] = (-1)^n x[n]        =>  DFT(x')[s] = X[s ^ N/2]      (input flip)
//   y[s]  = x[s ^ N/2]         =>  DFT(y)[k]  = (-1)^k DFT(x)[k] (output flip)
// so a thread with b = 1 negates its odd inputs before the first DFT and its
// odd outputs after the last one; nothing else changes.  (N1 = N2 only.)
//
// Modes (Eq. 12; the multiplier is the Fourier symbol of
// (L+1)^-1 with 1/N_vox folded in):
//   S_FWD          y forward                       (K_B)
//   S_INV          y inverse  = conj(DFT(conj(.))) (K_D)
//   S_FWD_MUL_INV  z (or 2-D y) forward, x g(p), inverse (K_C)
// The inverse is always computed as conj(DFT(conj(.))) so ONE FFT body is
// compiled per kernel (the unrolled body of two would overflow the I-cache).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "stile_core.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

// ZP (K_C on the z-pair layout of work, usp_internal.h WLayout): the tile's
// N z-rows of 16 columns are N/2 pair rows of 32 columns (16 x of planes 2zp
// and 2zp + 1 side by side), loaded as {32, BP} boxes and stored as 256-byte
// rows; the FFT, the multiplier and the exchange are unchanged.
template <int N, int MODE, bool ZP = false>
__global__ void __launch_bounds__(STile<N>::NT, STile<N>::MINB)
    k_stile(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap smap, SParams p) {
    using G = LineGeo<N>;
    using T = STile<N>;
    static_assert(!ZP || (MODE == S_FWD_MUL_INV && T::COLS == 16 && G::N1 % 2 == 0), "z-pair tiles: K_C, N <= 1024");
    constexpr int BP = (N / 4 < 256) ? N / 4 : 256;   // pair rows per box
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int g = tid / T::NTG, tl = tid % T::NTG;     // thread group, thread in group
    float2 *stage = reinterpret_cast<float2 *>(smem_raw) + g * T::GSM;
    float2 *xb = stage + T::TILE;
    float2 *sm_tw = reinterpret_cast<float2 *>(smem_raw) + T::GROUPS * T::GSM;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N) + g;
    const int bar = 1 + g;
    pdl_trigger();
    if (tid == 0) prefetch_tmap(&tmap);
    pdl_wait();
    if (p.check_state && !iter_running(p.st)) return;
    const int c = tl % T::COLS, j = tl / T::COLS;
    const long long tpo = p.ncols / T::COLS;
    const long long ntiles = tpo * p.nouter;
    // tiles are dealt to (CTA, group) pairs round-robin
    const long long vb = (long long)blockIdx.x * T::GROUPS + g, vg = (long long)gridDim.x * T::GROUPS;
    const int nloc = (int)((ntiles - vb + vg - 1) / vg);

    auto issue = [&](int i) {   // thread 0 of the group: TMA boxes of local tile i
        const long long t = vb + (long long)i * vg;
        const long long ol = t / tpo, o = ol;
        const int c0 = (int)((t - ol * tpo) * T::COLS);
        mbar_arrive_expect_tx(full, T::TILE * 8);
        if constexpr (ZP) {
#pragma unroll
            for (int bx = 0; bx < N / 2 / BP; ++bx) tma_load_2d(stage + bx * BP * 32, &tmap, (int)(t * 32), bx * BP, full);
        } else if (p.map_rank == 5) {
            // K_D after the return transpose: the line's rows live in P blocks of
            // the send layout [r][q][z_loc][y_loc][x] (5-D map {x, y_loc, z_loc, q, r})
            const int r = (int)(o / p.nz_loc), zl = (int)(o - (long long)r * p.nz_loc);
            const int lg = p.nyl_lg < ilog2(T::BOXN) ? p.nyl_lg : ilog2(T::BOXN);
            const int nyl_mask = (1 << p.nyl_lg) - 1;
            for (int y0 = 0; y0 < N; y0 += (1 << lg))
                tma_load_5d(stage + y0 * T::COLS, &tmap, c0, y0 & nyl_mask, zl, y0 >> p.nyl_lg, r, full);
        } else {
            // K_D on the z-pair buffer: plane o = half o & 1 of pair plane o >> 1 of the
            // [nz/2][ny][2 nx] view, its 16-column block at 32 (c0 / 16) + 16 (o & 1)
            const int cx = p.pair_src ? (c0 >> 4) * 32 + (int)(o & 1) * 16 : c0 + p.col0;
            const int ox = p.pair_src ? (int)(o >> 1) : (int)o;
#pragma unroll
            for (int bx = 0; bx < N / T::BOXN; ++bx) {
                if (p.map_rank == 3)
                    tma_load_3d(stage + bx * T::BOXN * T::COLS, &tmap, cx, bx * T::BOXN, ox, full);
                else tma_load_2d(stage + bx * T::BOXN * T::COLS, &tmap, c0 + p.col0, (int)o * N + bx * T::BOXN, full);
            }
        }
    };
    if (tl == 0) {
        prefetch_tmap(&tmap);
        mbar_init(full, 1);
        fence_mbar_init();
        if (nloc > 0) issue(0);
    }
    load_twiddles<N>(sm_tw, p.tw);
    __syncthreads();

    // FLIP shift flips: threads whose top row bit is set negate odd inputs /
    // outputs (see header).  The bit is uniform per warp (a warp holds the
    // rows 32/COLS consecutive j), so the flips are a non-divergent branch.
    const bool flip = T::FLIP && ((j >> (ilog2(G::N1) - 1)) & 1);
    // stashed tile rows [N - SROWS, N) = register slots m >= SM0 (see SParams::tma_store)
    constexpr int SROWS = T::HALFX ? N / 2 : N;
    constexpr int SM0 = T::HALFX ? G::N2 / 2 : 0;
    static_assert(!T::HALFX || T::XB >= (N / 2) * T::COLS, "stash needs half a tile");
    const bool TST = T::COLS == 16 && (ZP || SROWS >= T::BOXN) && p.tma_store;

    for (int i = 0; i < nloc; ++i) {
        if (!mbar_wait(full, i & 1)) {
            if (tl == 0 && atomicCAS(&p.st->err, 0, 5) == 0) p.st->err_info = i;
            return;
        }
        float2 v[G::N2];
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            // z-pair: plane z = j + N1 m sits in pair row z / 2, half z % 2
            const int z = j + G::N1 * m;
            const float2 a = ZP ? stage[(z >> 1) * 32 + (z & 1) * 16 + c] : stage[z * T::COLS + c];
            v[m] = (MODE == S_INV) ? cconj(a) : a;
        }
        if (flip) {
#pragma unroll
            for (int m = 1; m < G::N2; m += 2) v[m] = cscale(v[m], -1.f);
        }
        fence_proxy_async_smem();
        // the previous tile's stashed half must have left the exchange buffer
        // before anyone writes it again (first exchange of this tile)
        if (TST && tl == 0) bulk_wait_read0();
        gsync<N>(bar);                   // stage consumed: prefetch the next tile
        if (tl == 0 && i + 1 < nloc) issue(i + 1);

        if constexpr (MODE == S_FWD_MUL_INV) {
            float base;   // D (p_x^2 + p_y^2) + Re(sigma + c) of this thread's column
            {
                const long long t = vb + (long long)i * vg;
                const long long o = t / tpo;
                const long long col = (t - o * tpo) * T::COLS + c;
                float pt2;
                if (p.line_axis == 2) {
                    // column (x, y) of the (possibly y-sliced) z pass; y global
                    const long long gc = o * p.ncols + col;
                    const int ix = (int)(gc % p.mp.rowc) + p.x0, iy = (int)(p.y0 + gc / p.mp.rowc);
                    const float px = p.mp.kx * freq_m(ix, p.mp.nx), py = p.mp.ky * freq_m(iy, p.mp.ny);
                    pt2 = fmaf(px, px, py * py);
                } else {
                    const float px = p.mp.kx * freq_m((int)col, p.mp.nx);   // 2-D (complex path only)
                    pt2 = px * px;
                }
                base = fmaf(p.mp.D, pt2, p.mp.sc.x);
            }
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                stile_fft<N>(v, xb, sm_tw, c, j, bar);
                if (pass == 0) {
                    // (L+1)^-1 symbol (Eq. 12) at the signed frequency of k = j + N1 m:
                    //   g = cn (dr - i di) / (dr^2 + di^2),  dr = D |p|^2 + Re(sigma + c),
                    //   di = Im(sigma + c);  then conj so the second forward DFT inverts.
                    // (constants are re-derived here, opaque to hoisting, to keep them
                    // out of the registers live across the FFT)
                    // (kl is pre-scaled by sqrt(D): dr = (sqrt(D) p_line)^2 + base)
                    float di = p.mp.sc.y, kl = (p.line_axis == 2) ? p.mp.kz : p.mp.ky;
                    asm volatile("" : "+f"(di), "+f"(kl));
                    kl *= p.mp.sqrtD;
                    const float di2 = di * di, cyd = p.mp.cn.y * di, cxd = p.mp.cn.x * di;
                    const float klj = kl * (float)j;
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) {
                        const float cm = (float)(G::N1 * m - ((m >= G::N2 / 2) ? N : 0));
                        const float pl = fmaf(kl, cm, klj);
                        const float dr = fmaf(pl, pl, base);
                        const float inv = rcp_approx(fmaf(dr, dr, di2));
                        const float gr = fmaf(p.mp.cn.x, dr, cyd) * inv;
                        const float gi = fmaf(p.mp.cn.y, dr, -cxd) * inv;
                        v[m] = cconj(cmul(v[m], make_float2(gr, gi)));
                    }
                }
            }
        } else {
            stile_fft<N>(v, xb, sm_tw, c, j, bar);
        }
        long long t = vb + (long long)i * vg;
        asm volatile("" : "+l"(t));
        const long long ol = t / tpo, o = ol;
        const long long col = (t - ol * tpo) * T::COLS + c;
        long long stride = p.stride;
        asm volatile("" : "+l"(stride));
        if (flip) {
#pragma unroll
            for (int m = 1; m < G::N2; m += 2) v[m] = cscale(v[m], -1.f);
        }
        if constexpr (ZP) {
            // z-pair layout: register slot m = pair row (j >> 1) + (N1 / 2) m, half j & 1;
            // a warp (16 columns x 2 rows j) writes one 256-byte pair row per slot
            float2 *zb = p.dst + t * 32 + (j & 1) * 16 + c + (long long)(j >> 1) * stride;
            const long long zstep = (long long)(G::N1 / 2) * stride;
            if (TST) {
#pragma unroll
                for (int m = 0; m < SM0; ++m) zb[m * zstep] = cconj(v[m]);
#pragma unroll
                for (int m = SM0; m < G::N2; ++m)
                    xb[((j >> 1) + (G::N1 / 2) * m - (N - SROWS) / 2) * 32 + (j & 1) * 16 + c] = cconj(v[m]);
                fence_proxy_async_smem();
                gsync<N>(bar);
                if (tl == 0) {
#pragma unroll
                    for (int bx = 0; bx < SROWS / 2 / BP; ++bx)
                        tma_store_2d(&smap, (int)(t * 32), (N - SROWS) / 2 + bx * BP, xb + bx * BP * 32);
                    bulk_commit();
                }
            } else {
#pragma unroll
                for (int m = 0; m < G::N2; ++m) zb[m * zstep] = cconj(v[m]);
            }
        } else if (MODE == S_FWD && p.peer_mode == 1) {
            // K_B with the forward transpose fused in: row y of plane (r, z_loc)
            // is stored straight into block r of the receive buffer of rank
            // q = y / ny_loc ([z][y_loc][x] there) -- over NVLink for q != r
            const long long rr = o / p.nz_loc, zl = o - rr * p.nz_loc, r = p.rank0 + rr;
            const long long nyl = 1LL << p.nyl_lg;
            const long long off = r * p.bk + zl * nyl * p.ncols + col;
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const int y = j + G::N1 * m;
                p.peer[y >> p.nyl_lg][off + (long long)(y & (nyl - 1)) * stride] = v[m];
            }
        } else if (MODE == S_FWD_MUL_INV && p.peer_mode == 2) {
            // K_C with the return transpose fused in: z-line value z of y block r
            // goes to block r of the send buffer of the rank q = z / nz_loc that
            // owns plane z ([z_loc][y_loc][x] there); K_D reads it through the
            // 5-D map
            const long long off = (p.rank0 + o) * p.bk + col;
            const int zmask = p.nz_loc - 1, zlg = ilog2c(p.nz_loc);
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const int z = j + G::N1 * m;
                p.peer[z >> zlg][off + (long long)(z & zmask) * stride] = cconj(v[m]);
            }
        } else if (MODE == S_FWD && p.send_layout) {
            // K_B before the forward transpose: row y of plane o goes to block
            // (r, q = y / ny_loc) of the send layout [r][q][z_loc][y_loc][x]
            const long long r = o / p.nz_loc, zl = o - r * p.nz_loc;
            const long long nyl = 1LL << p.nyl_lg;
            const long long bk = (long long)p.nz_loc * nyl * p.ncols;
            float2 *sb = p.dst + r * p.P * bk + zl * nyl * p.ncols + col;
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const int y = j + G::N1 * m;
                sb[(y >> p.nyl_lg) * bk + (long long)(y & (nyl - 1)) * stride] = v[m];
            }
        } else if (TST) {
            // rows < N - SROWS straight from registers; rows >= N - SROWS into
            // the (free) exchange buffer as a dense [row][COLS] block, written
            // back by tensor-map stores while the next tile computes
            store_slots<N, MODE, 0, SM0>(v, p.dst + (o * p.ostride + col), stride, j, c);
#pragma unroll
            for (int m = SM0; m < G::N2; ++m)
                xb[(j + G::N1 * m - (N - SROWS)) * T::COLS + c] = (MODE == S_FWD) ? v[m] : cconj(v[m]);
            fence_proxy_async_smem();
            gsync<N>(bar);
            if (tl == 0) {
                const int c0 = (int)(col - c);
#pragma unroll
                for (int bx = 0; bx < SROWS / T::BOXN; ++bx) {
                    const int r0 = N - SROWS + bx * T::BOXN;
                    if (p.map_rank == 3) tma_store_3d(&smap, c0, r0, (int)o, xb + (r0 - (N - SROWS)) * T::COLS);
                    else tma_store_2d(&smap, c0, (int)o * N + r0, xb + (r0 - (N - SROWS)) * T::COLS);
                }
                bulk_commit();
            }
        } else {
            // K_B into the z-pair buffer: plane o -> pair plane o >> 1, half o & 1
            const long long ob = p.pair_dst ? (o >> 1) * p.ostride + (o & 1) * 16 + ((col >> 4) << 5) + (col & 15)
                                            : o * p.ostride + col;
            store_slots<N, MODE, 0, G::N2>(v, p.dst + ob, stride, j, c);
        }
    }
    if (TST && tl == 0) bulk_wait0();   // the exchange buffer outlives the last bulk store
    // fused transposes: this thread's stores into the peers' buffers (NVLink)
    // are performed at system scope before anything the GPU does after this
    // kernel -- in particular before the cross-rank barrier (an NCCL
    // collective on the same stream) that lets the peers read them
    if (p.peer_mode) __threadfence_system();
}

// ========================================================= launchers ====
template <int N, int MODE, bool ZP = false>
static cudaError_t stile_t(const CUtensorMap &map, const CUtensorMap &smap, const SParams &p, int grid,
                           cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(k_stile<N, MODE, ZP>, cudaFuncAttributeMaxDynamicSharedMemorySize, STile<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_pdl(k_stile<N, MODE, ZP>, grid, STile<N>::NT, STile<N>::SMEM, s, map, smap, p);
}

template <int N>
static cudaError_t stile_mode(SMode mode, const CUtensorMap &map, const CUtensorMap &smap, const SParams &p, int grid,
                              cudaStream_t s) {
    if (mode == S_FWD) return stile_t<N, S_FWD>(map, smap, p, grid, s);
    if (mode == S_INV) return stile_t<N, S_INV>(map, smap, p, grid, s);
    if (p.zpair) {
        if constexpr (N <= 1024) return stile_t<N, S_FWD_MUL_INV, true>(map, smap, p, grid, s);
        else return cudaErrorInvalidValue;
    }
    return stile_t<N, S_FWD_MUL_INV>(map, smap, p, grid, s);
}

bool stile_supported(long long n) { return n >= 64 && n <= 2048 && (n & (n - 1)) == 0; }
int stile_cols(int N) { return N == 2048 ? STile<2048>::COLS : (N == 1024 ? STile<1024>::COLS : 16); }
int stile_box(int N) { return N < 256 ? N : 256; }
int stile_ctas_per_sm(int N) {
    switch (N) {
    case 64: return STile<64>::MINB;
    case 128: return STile<128>::MINB;
    case 256: return STile<256>::MINB;
    case 512: return STile<512>::MINB;
    case 1024: return STile<1024>::MINB;
    case 2048: return STile<2048>::MINB;
    default: return 1;
    }
}

cudaError_t launch_stile(int N, SMode mode, const CUtensorMap &map, const CUtensorMap &smap, const SParams &p, int grid,
                         cudaStream_t s) {
    switch (N) {
    case 64: return stile_mode<64>(mode, map, smap, p, grid, s);
    case 128: return stile_mode<128>(mode, map, smap, p, grid, s);
    case 256: return stile_mode<256>(mode, map, smap, p, grid, s);
    case 512: return stile_mode<512>(mode, map, smap, p, grid, s);
    case 1024: return stile_mode<1024>(mode, map, smap, p, grid, s);
    case 2048: return stile_mode<2048>(mode, map, smap, p, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace usp
