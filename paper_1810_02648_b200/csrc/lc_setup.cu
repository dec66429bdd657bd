// Per-frame setup kernels: blur pyramid, mask contour + NN grid, two-pass
// rasterizer, FK / DQ skinning, occluding contour vertices, rim filter and
// body-part gating.  All batched over streams with blockIdx.y (or one CTA per
// stream where a CTA-wide ordered scan is needed).
#include <climits>
#include "lc_kernels.cuh"

// ===========================================================================
// separable Gaussian, mode "nearest" (scipy.ndimage.convolve1d order: centre
// tap first, then symmetric pairs from the outermost inward -- verified
// bit-exact against scipy 1.18.1).  imageproc.py:276-285

__global__ void k_blur_axis(JobArg<PyrJob> jobs, int H, int W, int C, const double *taps, int half,
                            int axis) {
    lc_pdl_wait();
    const PyrJob J = jobs[blockIdx.y];
    const double *in = axis == 0 ? J.src : J.tmp;
    double *out = axis == 0 ? J.tmp : J.dst;
    const long long n = (long long)H * W * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        const long long pix = i / C;
        const int x = (int)(pix % W), y = (int)(pix / W);
        double acc = in[i] * taps[half];
        if (axis == 0) {
            for (int j = half; j >= 1; --j) {
                const int ya = max(y - j, 0), yb = min(y + j, H - 1);
                acc = acc + (in[((long long)ya * W + x) * C + c] + in[((long long)yb * W + x) * C + c])
                                * taps[half + j];
            }
        } else {
            for (int j = half; j >= 1; --j) {
                const int xa = max(x - j, 0), xb = min(x + j, W - 1);
                acc = acc + (in[((long long)y * W + xa) * C + c] + in[((long long)y * W + xb) * C + c])
                                * taps[half + j];
            }
        }
        out[i] = acc;
    }
}

// One CTA per 32x32 output tile and stream: the haloed input tile is loaded
// once (coordinates clamped = mode "nearest"), then for every level the
// vertical pass fills a shared intermediate over the tile columns +- halo and
// the horizontal pass writes the level.  Each output is the same expression
// in the same order as the two-pass version, so results are bit-identical.
// shared memory: the haloed input tile (rows of 3E doubles, shifted by one
// double so interior rows load as 16-byte cp.async), the vertical pass's
// intermediate, and the output tile staged for coalesced 16-byte stores
// (the intermediate and the staged output have odd row strides, 3E + 1 and
// 3T + 1 doubles, so the horizontal pass -- one row per lane -- is free of
// bank conflicts)
#define LC_PYR_MS (3 * (LC_PYR_TILE + 2 * LC_PYR_HALO) + 1)
#define LC_PYR_OS (3 * LC_PYR_TILE + 1)
size_t pyramid_fused_smem() {
    const int T = LC_PYR_TILE, E = LC_PYR_TILE + 2 * LC_PYR_HALO;
    return sizeof(double) * ((size_t)E * (3 * E + 2) + (size_t)T * LC_PYR_MS + (size_t)T * LC_PYR_OS);
}

// Register-blocked passes: a thread owns RB consecutive outputs along the
// filter axis and loads its (RB + 2*HH)-wide window once.  Each output is
// still  w[c]*x[0] + (x[-h]+x[h])*w[h] + ... + (x[-1]+x[1])*w[1]  in that order.
template <int HH>
__device__ __forceinline__ void pyr_level(const double *__restrict__ in, double *__restrict__ mid,
                                          double *__restrict__ ot, double *__restrict__ out,
                                          const double *__restrict__ tp, int tx0, int ty0, int H, int W) {
    constexpr int T = LC_PYR_TILE, R = LC_PYR_HALO, E = T + 2 * R, RB = 8, NWIN = RB + 2 * HH;
    constexpr int SI = 3 * E + 2;   // input row stride (a padding double on either side)
    double t[HH + 1];
#pragma unroll
    for (int j = 0; j <= HH; ++j) t[j] = tp[HH + j];
    // vertical: unit = (tile column col in [0,3E), row block rb in [0,T/RB))
    for (int u = threadIdx.x; u < 3 * E * (T / RB); u += blockDim.x) {
        const int col = u % (3 * E), rb = u / (3 * E);
        const double *p = in + (rb * RB + R - HH) * SI + col;
        double win[NWIN];
#pragma unroll
        for (int k = 0; k < NWIN; ++k) win[k] = p[k * SI];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            double acc = win[r + HH] * t[0];
#pragma unroll
            for (int j = HH; j >= 1; --j) acc = acc + (win[r + HH - j] + win[r + HH + j]) * t[j];
            mid[(rb * RB + r) * LC_PYR_MS + col] = acc;
        }
    }
    __syncthreads();
    // horizontal: unit = (row, channel, column block), the row fastest (a
    // warp's lanes read / write 32 rows at odd strides); mid holds clamped columns
    for (int u = threadIdx.x; u < T * 3 * (T / RB); u += blockDim.x) {
        const int row = u % T, cc = u / T, c = cc % 3, cb = cc / 3;
        const int gy = ty0 + row;
        if (gy >= H) continue;
        const double *p = mid + row * LC_PYR_MS + (cb * RB + R - HH) * 3 + c;
        double win[NWIN];
#pragma unroll
        for (int k = 0; k < NWIN; ++k) win[k] = p[3 * k];
        double *o = ot + (size_t)row * LC_PYR_OS + (cb * RB) * 3 + c;   // the staged output tile
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            double acc = win[r + HH] * t[0];
#pragma unroll
            for (int j = HH; j >= 1; --j) acc = acc + (win[r + HH - j] + win[r + HH + j]) * t[j];
            o[3 * r] = acc;
        }
    }
    __syncthreads();
    // the tile's rows are 3T contiguous doubles in the level: 16-byte stores
    // when the row segment is whole and aligned, else element by element
    const int wx = min(T, W - tx0), hy = min(T, H - ty0);
    const bool vec = wx == T && ((((size_t)tx0 * 3) & 1) == 0) && ((((size_t)W * 3) & 1) == 0) &&
                     ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    if (vec) {
        constexpr int PR = 3 * T / 2;   // 16-byte pairs per row
        for (int q = threadIdx.x; q < hy * PR; q += blockDim.x) {
            const int row = q / PR, k = q - row * PR;
            double2 *dst = reinterpret_cast<double2 *>(out + ((size_t)(ty0 + row) * W + tx0) * 3);
            const double *src = ot + (size_t)row * LC_PYR_OS + 2 * k;
            dst[k] = make_double2(src[0], src[1]);
        }
    } else {
        for (int q = threadIdx.x; q < hy * 3 * wx; q += blockDim.x) {
            const int row = q / (3 * wx), k = q - row * 3 * wx;
            out[((size_t)(ty0 + row) * W + tx0) * 3 + k] = ot[(size_t)row * LC_PYR_OS + k];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_pyramid_fused(JobArg<PyrAllJob> jobs, int H, int W, int levels,
                                                       const double *taps, int h0, int h1, int h2, int h3) {
    lc_pdl_wait();
    const PyrAllJob J = jobs[blockIdx.y];
    constexpr int T = LC_PYR_TILE, R = LC_PYR_HALO, E = T + 2 * R;
    extern __shared__ double sm[];
    constexpr int SI = 3 * E + 2;        // input row stride: element -1 of every row is 16-byte aligned
    double *in = sm + 1;                 // E rows x SI
    double *mid = sm + E * SI;           // T rows x 3E (stride LC_PYR_MS)
    double *ot = mid + T * LC_PYR_MS;    // T rows x 3T (staged output, stride LC_PYR_OS)
    const int tiles_x = (W + T - 1) / T, ntiles = tiles_x * ((H + T - 1) / T);
    // grid-stride over the tiles (one tile per CTA at the default grid)
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx0 = (tile % tiles_x) * T, ty0 = (tile / tiles_x) * T;
    if (J.tile_flag) {   // region of interest (k_pyr_roi's flags): other tiles take the exact on-demand path
        if (J.roi) {
            if (!J.tile_flag[tile]) continue;
        } else if (threadIdx.x == 0) {
            J.tile_flag[tile] = 1;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // asynchronous tile copy (LDGSTS).  Interior tiles (no clamped column):
    // each row's 3E doubles start one double after a 16-byte boundary in both
    // the frame and shared memory, so the row moves as 16-byte copies of
    // elements [-1, 3E) (the extra leading double is harmless); tiles at the
    // left / right border clamp per element with 8-byte copies
    const bool interior = tx0 - R - 1 >= 0 && tx0 + T + R < W && (((size_t)W * 3) & 1) == 0 &&
                          ((((size_t)(tx0 - R) * 3) & 1) == 1) && ((reinterpret_cast<uintptr_t>(J.src) & 15) == 0);
    for (int row = warp; row < E; row += nw) {
        const int gy = min(max(ty0 + row - R, 0), H - 1);
        const double *src = J.src + (size_t)gy * W * 3;
        if (interior) {
            const double *s0 = src + (size_t)(tx0 - R) * 3 - 1;
            double *d0 = in + row * SI - 1;
            for (int k = lane; k < SI / 2; k += 32) {   // elements [-1, 3E + 1): the row's padding included
                const unsigned dst = (unsigned)__cvta_generic_to_shared(d0 + 2 * k);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(s0 + 2 * k));
            }
        } else {
            for (int col = lane; col < 3 * E; col += 32) {
                const int x = col / 3;
                const int gx = min(max(tx0 + x - R, 0), W - 1);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(in + row * SI + col);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                             "l"(src + gx * 3 + (col - 3 * x)));
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    const int hs[4] = {h0, h1, h2, h3};
    for (int l = 0; l < levels; ++l) {
        double *out = J.dst + (size_t)l * H * W * 3;
        const double *tp = taps + 32 * l;
        switch (hs[l]) {
            case 0: pyr_level<0>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 1: pyr_level<1>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 2: pyr_level<2>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 3: pyr_level<3>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 4: pyr_level<4>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 5: pyr_level<5>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            case 6: pyr_level<6>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
            default: pyr_level<7>(in, mid, ot, out, tp, tx0, ty0, H, W); break;
        }
    }
    }   // tiles (pyr_level ends with a block barrier: `in` is free for the next tile)
}

// One CTA per stream: the pyramid's region of interest.  The bounding box
// of the grid cells holding contour pixels (= the observed silhouette's),
// dilated by `margin` pixels, as a tile range; inside it, the tiles within
// ceil(margin / LC_PYR_TILE) tiles of a tile holding foreground (the
// per-row flags k_contour_rows leaves) get tile_flag = 1.  margin < 0: an
// empty region (every sample takes the exact on-demand path; a test hook).
#define LC_ROI_MAX_TILES 16384
__global__ void __launch_bounds__(1024) k_pyr_roi(JobArg<PyrRoiJob> jobs, int ncx, int ncy, int tiles_x,
                                                  int tiles_y, int margin, int H) {
    lc_pdl_wait();
    const PyrRoiJob J = jobs[blockIdx.x];
    __shared__ int b[4];
    __shared__ int r[4];
    __shared__ uint8_t fg[LC_ROI_MAX_TILES];
    if (threadIdx.x == 0) { b[0] = INT_MAX; b[1] = INT_MAX; b[2] = -1; b[3] = -1; }
    __syncthreads();
    int x0 = INT_MAX, y0 = INT_MAX, x1 = -1, y1 = -1;
    for (int i = threadIdx.x; i < ncx * ncy; i += blockDim.x)
        if (J.cell_count[i] > 0) {
            const int cx = i % ncx, cy = i / ncx;
            x0 = min(x0, cx); x1 = max(x1, cx); y0 = min(y0, cy); y1 = max(y1, cy);
        }
    if (x1 >= 0) {
        atomicMin(&b[0], x0); atomicMin(&b[1], y0); atomicMax(&b[2], x1); atomicMax(&b[3], y1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int q[4] = {1, 1, 0, 0};   // empty
        if (b[2] >= 0 && margin >= 0) {
            const int px0 = b[0] * LC_GRID_CELL - margin, py0 = b[1] * LC_GRID_CELL - margin;
            const int px1 = (b[2] + 1) * LC_GRID_CELL - 1 + margin, py1 = (b[3] + 1) * LC_GRID_CELL - 1 + margin;
            q[0] = max(0, px0) / LC_PYR_TILE;
            q[1] = max(0, py0) / LC_PYR_TILE;
            q[2] = min(tiles_x - 1, px1 / LC_PYR_TILE);
            q[3] = min(tiles_y - 1, py1 / LC_PYR_TILE);
        }
        for (int k = 0; k < 4; ++k) { J.roi[k] = q[k]; r[k] = q[k]; }
    }
    __syncthreads();
    if (!J.tile_flag) return;
    const int nt = tiles_x * tiles_y;
    const bool fine = J.fg_rows && nt <= LC_ROI_MAX_TILES;   // else the whole box
    if (fine)
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {
            const int tx = t % tiles_x, ty = t / tiles_x;
            uint8_t any = 0;
            for (int y = ty * LC_PYR_TILE; y < min(H, (ty + 1) * LC_PYR_TILE); ++y) any |= J.fg_rows[(size_t)y * tiles_x + tx];
            fg[t] = any;
        }
    __syncthreads();
    const int d = margin >= 0 ? (margin + LC_PYR_TILE - 1) / LC_PYR_TILE : 0;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const int tx = t % tiles_x, ty = t / tiles_x;
        bool want = tx >= r[0] && tx <= r[2] && ty >= r[1] && ty <= r[3];
        if (want && fine) {
            bool near = false;
            for (int yy = max(0, ty - d); yy <= min(tiles_y - 1, ty + d) && !near; ++yy)
                for (int xx = max(0, tx - d); xx <= min(tiles_x - 1, tx + d); ++xx)
                    if (fg[yy * tiles_x + xx]) { near = true; break; }
            want = near;
        }
        J.tile_flag[t] = want ? 1 : 0;
    }
}

// ===========================================================================
// contour pixels of a mask in np.argwhere (row-major) order, then a uniform
// cell grid over them.  imageproc.py:34-49

__device__ __forceinline__ bool is_contour(const uint8_t *m, int H, int W, int x, int y) {
    if (!m[y * W + x]) return false;
    const bool up = y > 0 && m[(y - 1) * W + x];
    const bool dn = y < H - 1 && m[(y + 1) * W + x];
    const bool lf = x > 0 && m[y * W + x - 1];
    const bool rt = x < W - 1 && m[y * W + x + 1];
    return !(up && dn && lf && rt);
}

// one block per row: row_count[y]
__global__ void k_contour_rows(JobArg<GridJob> jobs, int H, int W) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.y];
    __shared__ int cnt;
    for (int y = blockIdx.x; y < H; y += gridDim.x) {
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        int local = 0;
        for (int x = threadIdx.x; x < W; x += blockDim.x) local += is_contour(J.mask, H, W, x, y);
        if (J.fg_rows)   // foreground per LC_PYR_TILE-px segment of the row (for the pyramid's region of interest)
            for (int x0 = (threadIdx.x >> 5) * 32; x0 < W; x0 += blockDim.x) {
                const int x = x0 + (threadIdx.x & 31);
                const bool f = __any_sync(0xffffffffu, x < W && J.mask[(size_t)y * W + x] != 0);
                if ((threadIdx.x & 31) == 0) J.fg_rows[(size_t)y * ((W + LC_PYR_TILE - 1) / LC_PYR_TILE) + x0 / LC_PYR_TILE] = f;
            }
        for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&cnt, local);
        __syncthreads();
        if (threadIdx.x == 0) J.row_count[y] = cnt;
        __syncthreads();
    }
}

// block-wide exclusive scan of n ints (single CTA); returns the total
template <int NT>
__device__ int block_exclusive_scan(const int *in, int *out, int n) {
    __shared__ int warp_tot[NT / 32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += NT) {
        const int i = base + threadIdx.x;
        const int v = i < n ? in[i] : 0;
        int s = v;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        if (lane == 31) warp_tot[w] = s;
        __syncthreads();
        if (w == 0) {
            int t = lane < NT / 32 ? warp_tot[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            if (lane < NT / 32) warp_tot[lane] = t;
        }
        __syncthreads();
        const int before = (w > 0 ? warp_tot[w - 1] : 0) + carry;
        if (i < n) out[i] = before + s - v;
        __syncthreads();
        if (threadIdx.x == NT - 1) carry = before + s;
        __syncthreads();
    }
    return carry;
}

__global__ void k_contour_scan_rows(JobArg<GridJob> jobs, int H, int ncells) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.x];
    const int total = block_exclusive_scan<1024>(J.row_count, J.row_start, H);
    if (threadIdx.x == 0) {
        J.row_start[H] = total;
        *J.K = total;
    }
    for (int c = threadIdx.x; c < ncells; c += blockDim.x) {
        J.cell_count[c] = 0;
        J.cell_fill[c] = 0;
    }
}

// one block per row: ordered emission of (x, y) + per-cell counts
__global__ void k_contour_emit(JobArg<GridJob> jobs, int H, int W, int ncx) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.y];
    __shared__ int wsum[32];
    __shared__ int carry;
    for (int y = blockIdx.x; y < H; y += gridDim.x) {
        if (threadIdx.x == 0) carry = J.row_start[y];
        __syncthreads();
        for (int base = 0; base < W; base += blockDim.x) {
            const int x = base + threadIdx.x;
            const bool f = x < W && is_contour(J.mask, H, W, x, y);
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            if (lane == 0) wsum[w] = __popc(bal);
            __syncthreads();
            int before = carry;
            for (int k = 0; k < w; ++k) before += wsum[k];
            if (f) {
                const int slot = before + __popc(bal & ((1u << lane) - 1u));
                J.pts[slot] = make_int2(x, y);
                atomicAdd(&J.cell_count[(y >> LC_GRID_SHIFT) * ncx + (x >> LC_GRID_SHIFT)], 1);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int t = 0;
                for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += wsum[k];
                carry += t;
            }
            __syncthreads();
        }
    }
}

__global__ void k_contour_scan_cells(JobArg<GridJob> jobs, int ncells) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.x];
    const int total = block_exclusive_scan<1024>(J.cell_count, J.cell_start, ncells);
    if (threadIdx.x == 0) J.cell_start[ncells] = total;
}

__global__ void k_contour_fill(JobArg<GridJob> jobs, int ncx) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.y];
    const int K = *J.K;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
        const int2 p = J.pts[k];
        const int c = (p.y >> LC_GRID_SHIFT) * ncx + (p.x >> LC_GRID_SHIFT);
        const int s = atomicAdd(&J.cell_fill[c], 1);
        J.cell_pts[J.cell_start[c] + s] = k;
    }
}

// ---- site-count quadtree over the cells (one CTA per stream) -------------
__global__ void k_quad_build(JobArg<GridJob> jobs, int ncx, int ncy) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.x];
    const int P = J.qP;
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
        const int cx = i % P, cy = i / P;
        J.quad[i] = (cx < ncx && cy < ncy) ? J.cell_count[cy * ncx + cx] : 0;
    }
    __syncthreads();
    for (int l = 1; l <= J.qL; ++l) {
        const int side = P >> l, cside = side * 2;
        const int o = quad_off(P, l), co = quad_off(P, l - 1);
        for (int i = threadIdx.x; i < side * side; i += blockDim.x) {
            const int x = i % side, y = i / side;
            const int *c = J.quad + co;
            J.quad[o + i] = c[(2 * y) * cside + 2 * x] + c[(2 * y) * cside + 2 * x + 1]
                          + c[(2 * y + 1) * cside + 2 * x] + c[(2 * y + 1) * cside + 2 * x + 1];
        }
        __syncthreads();
    }
}

// ---- exact per-cell candidate lists (see NnGridDev) -----------------------

__device__ __forceinline__ NnGridDev grid_of(const GridJob &J, int H, int W) {
    NnGridDev g{};
    g.K = *J.K;
    g.W = W; g.H = H;
    g.ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL;
    g.ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
    g.pts = J.pts; g.cell_start = J.cell_start; g.cell_pts = J.cell_pts;
    g.quad = J.quad; g.qP = J.qP; g.qL = J.qL;
    return g;
}

// Per-cell candidate sets from the site-count quadtree (thread per cell).
// U2 = min over sites of the squared distance from the cell's farthest point;
// candidates = sites whose squared distance to the cell is <= U2.  Any query
// inside the cell has its nearest site (and every site tied with it) in the set.
struct CellBox { double x0, y0, x1, y1; };

__device__ __forceinline__ double near2_box(const CellBox &c, double bx0, double by0, double bx1, double by1) {
    const double dx = fmax(0.0, fmax(bx0 - c.x1, c.x0 - bx1));
    const double dy = fmax(0.0, fmax(by0 - c.y1, c.y0 - by1));
    return dx * dx + dy * dy;
}

// Warp-cooperative walk of the site quadtree: the traversal is warp-uniform
// (node tests use warp-uniform bounds), the sites of each visited leaf are
// split over the lanes: leaf(k0) is called by every lane, which handles
// sites k0 + lane, k0 + lane + 32, ...; `after_leaf()` re-synchronizes bounds.
template <typename K, typename L, typename A>
__device__ __forceinline__ void quad_walk_warp(const NnGridDev &g, const CellBox &cb, K &&keep, L &&leaf,
                                               A &&after_leaf) {
    int stack[3 * 12 + 2];
    int sp = 0;
    stack[sp++] = g.qL << 24;
    while (sp > 0) {
        const int e = stack[--sp];
        const int l = e >> 24, ny = (e >> 12) & 0xfff, nx = e & 0xfff;
        const int side = g.qP >> l;
        if (g.quad[quad_off(g.qP, l) + ny * side + nx] == 0) continue;
        const double s = (double)(LC_GRID_CELL << l);
        if (!keep(near2_box(cb, nx * s, ny * s, nx * s + s - 1.0, ny * s + s - 1.0))) continue;
        if (l == 0) {
            if (nx < g.ncx && ny < g.ncy) {
                const int c = ny * g.ncx + nx;
                leaf(g.cell_start[c], g.cell_start[c + 1]);
                after_leaf();
            }
            continue;
        }
        int ch[4];
        double d[4];
        const double cs = s * 0.5;
        for (int k = 0; k < 4; ++k) {
            const int cx = 2 * nx + (k & 1), cy = 2 * ny + (k >> 1);
            ch[k] = ((l - 1) << 24) | (cy << 12) | cx;
            d[k] = near2_box(cb, cx * cs, cy * cs, cx * cs + cs - 1.0, cy * cs + cs - 1.0);
        }
        for (int i = 1; i < 4; ++i)
            for (int j = i; j > 0 && d[j] > d[j - 1]; --j) {
                const double td = d[j]; d[j] = d[j - 1]; d[j - 1] = td;
                const int tc = ch[j]; ch[j] = ch[j - 1]; ch[j - 1] = tc;
            }
        for (int k = 0; k < 4; ++k) stack[sp++] = ch[k];
    }
}

__device__ __forceinline__ CellBox cell_box(int cx, int cy) {
    return CellBox{(double)(cx * LC_GRID_CELL), (double)(cy * LC_GRID_CELL),
                   (double)(cx * LC_GRID_CELL + LC_GRID_CELL), (double)(cy * LC_GRID_CELL + LC_GRID_CELL)};
}

// Jump flooding over the cell grid (one CTA per stream): every cell gets a
// site near its centre.  Only used as an upper bound for the candidate band
// (any real site bounds the nearest distance), so JFA's rare misses cost
// list length, never exactness.
__global__ void k_cell_jfa(JobArg<GridJob> jobs, int ncx, int ncy) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.x];
    extern __shared__ int seeds[];   // 2 * ncells ping-pong
    const int nc = ncx * ncy;
    int *a = seeds, *b = seeds + nc;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const int s0 = J.cell_start[c], s1 = J.cell_start[c + 1];
        a[c] = s1 > s0 ? J.cell_pts[s0] : -1;
    }
    __syncthreads();
    int step = 1;
    while (step * 2 < max(ncx, ncy)) step *= 2;
    auto pass = [&](int k) {
        for (int c = threadIdx.x; c < nc; c += blockDim.x) {
            const int cx = c % ncx, cy = c / ncx;
            const double qx = cx * LC_GRID_CELL + 0.5 * LC_GRID_CELL, qy = cy * LC_GRID_CELL + 0.5 * LC_GRID_CELL;
            int best = a[c];
            double bd = LC_INF;
            if (best >= 0) {
                const int2 p = J.pts[best];
                bd = (qx - p.x) * (qx - p.x) + (qy - p.y) * (qy - p.y);
            }
            for (int dy = -k; dy <= k; dy += k)
                for (int dx = -k; dx <= k; dx += k) {
                    const int nx = cx + dx, ny = cy + dy;
                    if ((dx == 0 && dy == 0) || nx < 0 || ny < 0 || nx >= ncx || ny >= ncy) continue;
                    const int sd = a[ny * ncx + nx];
                    if (sd < 0) continue;
                    const int2 p = J.pts[sd];
                    const double d = (qx - p.x) * (qx - p.x) + (qy - p.y) * (qy - p.y);
                    if (d < bd) { bd = d; best = sd; }
                }
            b[c] = best;
        }
        __syncthreads();
        int *t = a; a = b; b = t;
    };
    for (int k = step; k >= 1; k >>= 1) pass(k);
    pass(1);
    pass(1);
    for (int c = threadIdx.x; c < nc; c += blockDim.x) J.cell_seed[c] = a[c];
}

// warp per cell: bound U^2 (warp min), then the candidate count (warp sum)
// Exact per-cell candidate sets from the site-count quadtree, one warp per
// cell, in a single pass.  U2 bounds the cell's farthest-point nearest
// distance (via the jump-flooded seed); the candidates are the sites whose
// squared distance to the cell is <= U2, so any query inside the cell has
// its nearest site (and every site tied with it) among them.  The warp
// collects the keys (near2 << 32 | id) in shared memory while walking the
// quadtree, sorts them (bitonic network) by (distance to the cell, key) and
// writes the cell's fixed-capacity list (LC_CAND_MAX slots) and its 128 B
// block {start, count, first LC_CAND_HEAD keys}.  A query scans the list in
// that order and stops at the first entry farther from the cell than its
// best distance (nn_query), so only the head is read.  Cells with more than
// LC_CAND_MAX candidates (or beyond max_u2) keep the quadtree search.
#ifndef LC_DOMINATORS
#define LC_DOMINATORS 16
#endif
#ifndef LC_SEED_PRUNE
#define LC_SEED_PRUNE 1
#endif
// breadth-first candidate collection (0: the depth-first walk only);
// frontiers / leaf lists beyond LC_BFS_CAP nodes fall back to the walk
#ifndef LC_CAND_BFS
#define LC_CAND_BFS 1
#endif
#define LC_BFS_CAP 256
// Site s = (px, py) is dominated over the closed 16-px cell at (X0, Y0) by
// site t when |q-s|^2 - |q-t|^2 >= 1 at every point q of the cell: the
// difference is affine in q, so its minimum over the cell is at a corner,
// f(X0, Y0) + min(0, 16 a) + min(0, 16 b).  Exact integer arithmetic (I =
// int while every coordinate is below 8192, else long long); t == s gives 0.
template <typename I>
__device__ __forceinline__ bool cell_dominated(int tx, int ty, I t2, int px, int py, I s2, int X0, int Y0) {
    const I a = (I)(2 * (tx - px)), b = (I)(2 * (ty - py));
    const I f = a * X0 + b * Y0 + (s2 - t2) + min((I)0, a * LC_GRID_CELL) + min((I)0, b * LC_GRID_CELL);
    return f >= 1;
}

__global__ void __launch_bounds__(128) k_cand_build(JobArg<GridJob> jobs, int H, int W) {
    lc_pdl_wait();
    const GridJob J = jobs[blockIdx.y];
    const NnGridDev g = grid_of(J, H, W);
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    __shared__ unsigned long long keys_all[4][LC_CAND_MAX];
    __shared__ int bfs_all[4][2][LC_BFS_CAP];
    __shared__ int leaf_all[4][LC_BFS_CAP];
    unsigned long long *key = keys_all[threadIdx.x >> 5];
    for (int c = blockIdx.x * wpb + (threadIdx.x >> 5); c < g.ncx * g.ncy; c += gridDim.x * wpb) {
        const int cx = c % g.ncx, cy = c / g.ncx;
        const int start = c * LC_CAND_MAX;
        int n = 0;
        bool ok = g.K > 0;
        double u2 = LC_INF;
        if (ok) {
            const int seed = J.cell_seed[c];
            u2 = seed >= 0 ? cell_far2(cx, cy, g.pts[seed]) : LC_INF;
            ok = u2 <= J.max_u2;
        }
        // the jump-flooded seed (a real site near the cell) already dominates
        // most far candidates: drop them while collecting, so the sort and
        // the full dominance pass below see short lists (same exactness
        // argument as the dominance pruning: |q-s|^2 - |q-t|^2 >= 1 over the
        // whole cell means s is never the nearest, nor tied with it)
        const int X0 = cx * LC_GRID_CELL, Y0 = cy * LC_GRID_CELL;
        int2 sd = make_int2(0, 0);
        bool has_sd = false;
        if (ok && LC_SEED_PRUNE) {
            const int seed = J.cell_seed[c];
            if (seed >= 0) { sd = g.pts[seed]; has_sd = true; }
        }
        const bool small = W <= 8192 && H <= 8192;   // int32 dominance tests cannot overflow
        auto seed_dominates = [&](int2 p) {
            if (!has_sd) return false;
            if (small)
                return cell_dominated<int>(sd.x, sd.y, sd.x * sd.x + sd.y * sd.y, p.x, p.y, p.x * p.x + p.y * p.y,
                                           X0, Y0);
            return cell_dominated<long long>(sd.x, sd.y, (long long)sd.x * sd.x + (long long)sd.y * sd.y, p.x, p.y,
                                             (long long)p.x * p.x + (long long)p.y * p.y, X0, Y0);
        };
        // collect the candidates: the sites within u2 of the cell that the
        // seed does not dominate (appended in any order: the list is sorted
        // by (distance, key) below, so the visit order does not matter)
        auto consider = [&](int kk, bool valid) {
            bool take = false;
            int pid = 0;
            int2 p = make_int2(0, 0);
            if (valid) {
                pid = g.cell_pts[kk];
                p = g.pts[pid];
                take = cell_near2(cx, cy, p) <= u2 && !seed_dominates(p);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, take);
            const int at = n + __popc(bal & ((1u << lane) - 1u));
            if (take && at < LC_CAND_MAX)
                key[at] = ((unsigned long long)cell_near2_int(cx, cy, p) << 32) | (unsigned)pid;
            n += __popc(bal);
        };
        bool walked = false;
        if (ok && LC_CAND_BFS) {
            // breadth-first over the site quadtree, the lanes testing one
            // frontier node each (the same node set as the depth-first walk:
            // every non-empty node with near2 <= u2), then the sites of all
            // reached leaf cells flattened over the lanes, so the dependent
            // loads (node count; leaf range -> site id -> site) issue a warp
            // at a time instead of one node / one leaf at a time
            int *fr0 = bfs_all[threadIdx.x >> 5][0], *fr1 = bfs_all[threadIdx.x >> 5][1];
            int *leaf = leaf_all[threadIdx.x >> 5];
            const CellBox cb = cell_box(cx, cy);
            if (lane == 0) fr0[0] = g.qL << 24;
            __syncwarp();
            int nf = 1, nleaf = 0;
            bool over = false;
            while (nf > 0) {
                int nn = 0;
                for (int b = 0; b < nf; b += 32) {
                    const int i = b + lane;
                    bool inner = false, isleaf = false;
                    int l = 0, ny = 0, nx = 0;
                    if (i < nf) {
                        const int e = fr0[i];
                        l = e >> 24; ny = (e >> 12) & 0xfff; nx = e & 0xfff;
                        const int side = g.qP >> l;
                        if (g.quad[quad_off(g.qP, l) + ny * side + nx] != 0) {
                            const double sz = (double)(LC_GRID_CELL << l);
                            if (near2_box(cb, nx * sz, ny * sz, nx * sz + sz - 1.0, ny * sz + sz - 1.0) <= u2) {
                                if (l > 0) inner = true;
                                else isleaf = nx < g.ncx && ny < g.ncy;
                            }
                        }
                    }
                    const unsigned lt = (1u << lane) - 1u;
                    const unsigned bi = __ballot_sync(0xffffffffu, inner);
                    const int at = nn + 4 * __popc(bi & lt);
                    if (inner && at + 4 <= LC_BFS_CAP)
                        for (int k = 0; k < 4; ++k)
                            fr1[at + k] = ((l - 1) << 24) | ((2 * ny + (k >> 1)) << 12) | (2 * nx + (k & 1));
                    nn += 4 * __popc(bi);
                    const unsigned bl = __ballot_sync(0xffffffffu, isleaf);
                    const int al = nleaf + __popc(bl & lt);
                    if (isleaf && al < LC_BFS_CAP) leaf[al] = ny * g.ncx + nx;
                    nleaf += __popc(bl);
                }
                __syncwarp();
                if (nn > LC_BFS_CAP || nleaf > LC_BFS_CAP) { over = true; break; }
                int *t = fr0; fr0 = fr1; fr1 = t;
                nf = nn;
            }
            if (!over) {
                walked = true;
                // sites of the reached leaves, 32 leaves' ranges at a time
                for (int lb = 0; lb < nleaf; lb += 32) {
                    const int li = lb + lane;
                    int s0 = 0, cntl = 0;
                    if (li < nleaf) {
                        const int cc = leaf[li];
                        s0 = g.cell_start[cc];
                        cntl = g.cell_start[cc + 1] - s0;
                    }
                    int incl = cntl;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const int total = __shfl_sync(0xffffffffu, incl, 31);
                    int *excl = fr1;   // the frontier buffers are free now
                    int *sbase = fr0;
                    excl[lane] = incl - cntl;
                    sbase[lane] = s0;
                    __syncwarp();
                    const int nl = min(32, nleaf - lb);
                    for (int t0 = 0; t0 < total; t0 += 32) {
                        const int t = t0 + lane;
                        int kk = 0;
                        if (t < total) {
                            int lo = 0, hi = nl - 1;   // the last leaf whose start <= t
                            while (lo < hi) {
                                const int m = (lo + hi + 1) >> 1;
                                if (excl[m] <= t) lo = m; else hi = m - 1;
                            }
                            kk = sbase[lo] + (t - excl[lo]);
                        }
                        consider(kk, t < total);
                    }
                    __syncwarp();
                }
            }
        }
        if (ok && !walked)
            quad_walk_warp(g, cell_box(cx, cy), [&](double n2) { return n2 <= u2; },
                           [&](int k0, int k1) {
                               for (int k = k0; k < k1; k += 32) consider(k + lane, k + lane < k1);
                           },
                           [&]() {});
        if (ok) ok = n <= LC_CAND_MAX;
        if (ok) {
            int P = 1;
            while (P < n) P <<= 1;
            if (P <= 32) {
                // one key per lane: the bitonic network over shuffles
                unsigned long long v = lane < n ? key[lane] : ~0ull;
#pragma unroll
                for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, j);
                        v = (((lane & j) == 0) == ((lane & k) == 0)) ? (v < o ? v : o) : (v < o ? o : v);
                    }
                __syncwarp();
                if (lane < n) key[lane] = v;
                __syncwarp();
            } else {
                for (int i = n + lane; i < P; i += 32) key[i] = ~0ull;
                __syncwarp();
                for (int k = 2; k <= P; k <<= 1)
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        for (int i = lane; i < P; i += 32) {
                            const int ixj = i ^ j;
                            if (ixj > i) {
                                const unsigned long long a = key[i], b = key[ixj];
                                if ((a > b) == ((i & k) == 0)) { key[i] = b; key[ixj] = a; }
                            }
                        }
                        __syncwarp();
                    }
            }
            // Dominance pruning.  A candidate s is dropped when one of the
            // cell's LC_DOMINATORS closest candidates t dominates it over the
            // cell (cell_dominated: |q-s|^2 - |q-t|^2 >= 1 on the whole cell,
            // far beyond the rounding of the fp64 squared distances, < 1e-7
            // px^2 here), so s is never the nearest site -- nor tied with it
            // -- for any query in the cell.  Exact; it removes most of a far
            // cell's list (the contour sites far along the contour from the
            // cell's nearest ones).
            const int nd = min(n, LC_DOMINATORS);
            int tx[LC_DOMINATORS], ty[LC_DOMINATORS];
#pragma unroll
            for (int d = 0; d < LC_DOMINATORS; ++d) {
                const int2 p = d < nd ? g.pts[(int)(unsigned)(key[d] & 0xffffffffu)] : make_int2(0, 0);
                tx[d] = p.x;
                ty[d] = p.y;
            }
            int m = 0;
            for (int base = 0; base < n; base += 32) {
                const int i = base + lane;
                bool keep = false;
                int k = 0;
                if (i < n) {
                    const int2 p = g.pts[(int)(unsigned)(key[i] & 0xffffffffu)];
                    k = site_key(p);
                    keep = true;
                    if (small) {
                        const int s2 = p.x * p.x + p.y * p.y;
#pragma unroll
                        for (int d = 0; d < LC_DOMINATORS; ++d) {
                            if (d >= nd) break;
                            if (cell_dominated<int>(tx[d], ty[d], tx[d] * tx[d] + ty[d] * ty[d], p.x, p.y, s2, X0, Y0)) {
                                keep = false;
                                break;
                            }
                        }
                    } else {
                        const long long s2 = (long long)p.x * p.x + (long long)p.y * p.y;
#pragma unroll
                        for (int d = 0; d < LC_DOMINATORS; ++d) {
                            if (d >= nd) break;
                            if (cell_dominated<long long>(tx[d], ty[d], (long long)tx[d] * tx[d] + (long long)ty[d] * ty[d],
                                                          p.x, p.y, s2, X0, Y0)) {
                                keep = false;
                                break;
                            }
                        }
                    }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int pos = m + __popc(bal & ((1u << lane) - 1u));
                    J.cand_pts[start + pos] = k;
                    if (pos < LC_CAND_HEAD) J.cand_blk[32 * (size_t)c + 2 + pos] = k;
                }
                m += __popc(bal);
            }
            n = m;
        }
        if (lane == 0) {
            J.cand_blk[32 * (size_t)c] = start;
            J.cand_blk[32 * (size_t)c + 1] = ok ? n : -1;
        }
        __syncwarp();
    }
}

// ===========================================================================
// rasterizer.  The reference draws triangles sequentially and keeps the first
// strictly-smaller depth (rasterizer.py:46-58).  Pass 1 finds the minimum
// depth per pixel (atomicMin on the fp64 bit pattern: depths are positive);
// pass 2 picks the lowest triangle index attaining it; the resolve pass
// recomputes that triangle's barycentrics.  Same arithmetic, same order.

__device__ __forceinline__ bool tri_setup(CamDev cam, const double *V, const int *tris, int t,
                                          double P[3][2], double D[3], double &inv, int bb[4]) {
    const int ids[3] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    for (int k = 0; k < 3; ++k) {
        const V3 p = ld3(V + 3 * (size_t)ids[k]);
        double px, py;
        const bool ok = project(cam, p, px, py);
        P[k][0] = px;
        P[k][1] = py;
        D[k] = ok ? p.z : -1.0;
    }
    if (D[0] <= 0.0 || D[1] <= 0.0 || D[2] <= 0.0) return false;
    const double area = (P[1][0] - P[0][0]) * (P[2][1] - P[0][1]) - (P[2][0] - P[0][0]) * (P[1][1] - P[0][1]);
    if (area > -1e-12 && area < 1e-12) return false;
    inv = 1.0 / area;
    const double lx = fmin(P[0][0], fmin(P[1][0], P[2][0])), hx = fmax(P[0][0], fmax(P[1][0], P[2][0]));
    const double ly = fmin(P[0][1], fmin(P[1][1], P[2][1])), hy = fmax(P[0][1], fmax(P[1][1], P[2][1]));
    double x0 = floor(lx), x1 = ceil(hx), y0 = floor(ly), y1 = ceil(hy);
    x0 = fmax(x0, 0.0); y0 = fmax(y0, 0.0);
    x1 = fmin(x1, (double)(cam.W - 1)); y1 = fmin(y1, (double)(cam.H - 1));
    if (!(x0 <= x1 && y0 <= y1)) return false;
    bb[0] = (int)x0; bb[1] = (int)x1; bb[2] = (int)y0; bb[3] = (int)y1;
    return true;
}

__device__ __forceinline__ bool bary(const double P[3][2], double inv, int ix, int iy, double &l0,
                                     double &l1, double &l2) {
    const double px = (double)ix, py = (double)iy;
    l0 = ((P[1][0] - px) * (P[2][1] - py) - (P[2][0] - px) * (P[1][1] - py)) * inv;
    l1 = ((px - P[0][0]) * (P[2][1] - P[0][1]) - (P[2][0] - P[0][0]) * (py - P[0][1])) * inv;
    l2 = 1.0 - l0 - l1;
    return !(l0 < 0.0 || l1 < 0.0 || l2 < 0.0);
}

// Tile-binned single pass.  The sequential rule "first triangle with a
// strictly smaller depth wins" (rasterizer.py:46-58) leaves every pixel with
// the lexicographic minimum of (depth, triangle index) over the triangles
// covering it, so the order in which a tile meets its triangles does not
// matter.  Setup: one thread per triangle writes its TriRec (the reference's
// arithmetic: projection, signed area, clipped bbox).  Binning: one warp per
// triangle counts, then (after a per-stream scan) appends, the triangle in
// every tile of its bbox it can touch.  Resolve: one CTA per 16x16 tile
// stages the tile's triangles in shared memory and every thread resolves
// its pixel (depth, id and mask) in registers: no per-pixel atomics, no
// second pass, coalesced stores.  A tile whose list overflowed the buffer
// tests every triangle (still exact).

__global__ void k_rt_clear(JobArg<RasterJob> jobs, int n) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) J.tcount[i] = 0;
}

__global__ void k_rt_setup(JobArg<RasterJob> jobs, CamDev cam, const int *tris, int T) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    double P[3][2], D[3], inv = 0.0;
    int bb[4];
    const bool ok = tri_setup(cam, J.verts, tris, t, P, D, inv, bb);
    TriRec r;
    for (int k = 0; k < 3; ++k) {
        r.P[2 * k] = P[k][0];
        r.P[2 * k + 1] = P[k][1];
        r.D[k] = D[k];
    }
    r.inv = inv;
    if (ok) {
        for (int k = 0; k < 4; ++k) r.bb[k] = bb[k];
    } else {
        r.bb[0] = 1; r.bb[1] = 0; r.bb[2] = 1; r.bb[3] = 0;
    }
    J.rec[t] = r;
}

// Can triangle r cover a pixel of tile (tx, ty)?  No only when one
// barycentric coordinate is below -eps at all four corners of the tile's
// pixel box: the coordinate is affine, so every pixel of the tile then has
// it below -eps + 2 delta < 0 in the exact per-pixel test (delta bounds the
// rounding of bary's arithmetic; eps is set well above it).  This keeps
// slivers with huge bboxes (the reference's trackers produce them once they
// lose track) out of most tiles.
struct RtCull { double eps; bool on; };
__device__ __forceinline__ RtCull rt_cull(const TriRec &r, int ntiles) {
    double big = 2048.0;
    for (int k = 0; k < 6; ++k) big = fmax(big, fabs(r.P[k]));
    RtCull c;
    c.eps = 1e-3 + 64.0 * 2.220446049250313e-16 * (4.0 * big * big) * fabs(r.inv);
    c.on = ntiles > 1 && c.eps < 0.25;
    return c;
}
__device__ __forceinline__ bool rt_tile_hit(const TriRec &r, const int4 bb, RtCull c, int tx, int ty) {
    if (!c.on) return true;
    const double(*P)[2] = reinterpret_cast<const double(*)[2]>(r.P);
    const int x0 = max(tx << LC_RT_SHIFT, bb.x), x1 = min((tx << LC_RT_SHIFT) + LC_RT_TILE - 1, bb.y);
    const int y0 = max(ty << LC_RT_SHIFT, bb.z), y1 = min((ty << LC_RT_SHIFT) + LC_RT_TILE - 1, bb.w);
    bool out0 = true, out1 = true, out2 = true;
    const int cx[4] = {x0, x1, x0, x1}, cy[4] = {y0, y0, y1, y1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double l0, l1, l2;
        bary(P, r.inv, cx[q], cy[q], l0, l1, l2);
        out0 = out0 && l0 < -c.eps;
        out1 = out1 && l1 < -c.eps;
        out2 = out2 && l2 < -c.eps;
    }
    return !(out0 || out1 || out2);
}

// one warp per triangle over the tiles of its bbox: count (fill = 0) or append (fill = 1)
template <int FILL>
__global__ void k_rt_bin(JobArg<RasterJob> jobs, int T, int ntx) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= T) return;
    const TriRec &r = J.rec[t];
    const int4 bb = *reinterpret_cast<const int4 *>(r.bb);
    if (bb.x > bb.y) return;
    const int tx0 = bb.x >> LC_RT_SHIFT, tx1 = bb.y >> LC_RT_SHIFT;
    const int ty0 = bb.z >> LC_RT_SHIFT, ty1 = bb.w >> LC_RT_SHIFT;
    const int nx = tx1 - tx0 + 1, nt = nx * (ty1 - ty0 + 1);
    const RtCull c = rt_cull(r, nt);
    for (int k = lane; k < nt; k += 32) {
        const int ty = ty0 + k / nx, tx = tx0 + k % nx;
        if (!rt_tile_hit(r, bb, c, tx, ty)) continue;
        const int tile = ty * ntx + tx;
        if (FILL) {
            const int off = J.toff[tile] + atomicAdd(&J.tfill[tile], 1);
            if (off < J.tcap) J.tlist[off] = t;
        } else {
            atomicAdd(&J.tcount[tile], 1);
        }
    }
}
template __global__ void k_rt_bin<0>(JobArg<RasterJob>, int, int);
template __global__ void k_rt_bin<1>(JobArg<RasterJob>, int, int);

// block-wide exclusive scan of v(i), i < n, into out[i] (out[n] = total)
template <typename V>
__device__ void rt_block_scan(int n, V &&v, int *out, int *zero = nullptr) {
    __shared__ int wt[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int x = i < n ? v(i) : 0;
        int sc = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, sc, o);
            if (lane >= o) sc += u;
        }
        if (lane == 31) wt[w] = sc;
        __syncthreads();
        if (w == 0) {
            int u = lane < (int)(blockDim.x >> 5) ? wt[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int q = __shfl_up_sync(0xffffffffu, u, o);
                if (lane >= o) u += q;
            }
            if (lane < (int)(blockDim.x >> 5)) wt[lane] = u;
        }
        __syncthreads();
        const int before = (w > 0 ? wt[w - 1] : 0) + carry;
        if (i < n) {
            out[i] = before + sc - x;
            if (zero) zero[i] = 0;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = before + sc;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = carry;
    __syncthreads();
}

// Per stream (one CTA): list offsets from the per-tile counts, then work
// items: a tile's list is resolved in chunks of LC_RT_CHUNK triangles by
// separate CTAs (merged by k_rt_merge) so a tile that collects thousands of
// triangles (a collapsed, far-away surface) is still resolved in parallel.
// A tile whose list overflowed the buffer resolves every triangle in one CTA.
__global__ void k_rt_scan(JobArg<RasterJob> jobs, int n, int T) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.x];
    rt_block_scan(n, [&](int i) { return J.tcount[i]; }, J.toff, J.tfill);
    rt_block_scan(n, [&](int i) {
        if (J.toff[i + 1] > J.tcap) return 1;   // overflowed: one CTA over every triangle
        return max(1, (J.tcount[i] + LC_RT_CHUNK - 1) / LC_RT_CHUNK);
    }, J.ioff);
}

__device__ __forceinline__ void rt_pixel(const TriRec &r, int id, int x, int y, unsigned long long &zb, int &tb) {
    if (x < r.bb[0] || x > r.bb[1] || y < r.bb[2] || y > r.bb[3]) return;
    const double(*P)[2] = reinterpret_cast<const double(*)[2]>(r.P);
    double l0, l1, l2;
    if (!bary(P, r.inv, x, y, l0, l1, l2)) return;
    const double z = l0 * r.D[0] + l1 * r.D[1] + l2 * r.D[2];
    const unsigned long long bits = (unsigned long long)__double_as_longlong(z);   // z > 0
    if (bits < zb || (bits == zb && id < tb)) { zb = bits; tb = id; }
}

__device__ __forceinline__ void rt_write(const RasterJob &J, CamDev cam, int x, int y, unsigned long long zb, int tb) {
    if (x < cam.W && y < cam.H) {
        const size_t pi = (size_t)y * cam.W + x;
        J.zbuf[pi] = zb;
        J.tri_id[pi] = tb;
        if (J.mask) J.mask[pi] = zb != 0x7ff0000000000000ULL;
    }
}

// work items (tile, chunk), grid-strided; thread = pixel of the tile
__global__ void __launch_bounds__(256) k_rt_tiles(JobArg<RasterJob> jobs, CamDev cam, int T, int ntx, int nt) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    constexpr int CH = 64;
    __shared__ TriRec sr[CH];
    __shared__ int sid[CH];
    const int total = J.ioff[nt];
    const int extra = total - nt;   // items beyond one per tile (multi-chunk tiles)
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
        // the tile owning this item: last tile with ioff[tile] <= item.  Every
        // tile has at least one item, so tile <= ioff[tile] <= tile + extra:
        // the owner lies in [item - extra, item] (one probe when no tile is split)
        int lo = max(0, item - extra), hi = min(nt - 1, item);
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (J.ioff[mid] <= item) lo = mid;
            else hi = mid - 1;
        }
        const int tile = lo, chunk = item - J.ioff[tile], nchunks = J.ioff[tile + 1] - J.ioff[tile];
        const int x = (tile % ntx) * LC_RT_TILE + (threadIdx.x & (LC_RT_TILE - 1));
        const int y = (tile / ntx) * LC_RT_TILE + (threadIdx.x >> LC_RT_SHIFT);
        const bool all = J.toff[tile + 1] > J.tcap;   // overflowed list: every triangle (bbox-rejected cheaply)
        const int b0 = all ? 0 : J.toff[tile] + chunk * LC_RT_CHUNK;
        const int b1 = all ? T : min(J.toff[tile + 1], b0 + LC_RT_CHUNK);
        unsigned long long zb = 0x7ff0000000000000ULL;
        int tb = INT_MAX;
        for (int base = b0; base < b1; base += CH) {
            const int n = min(CH, b1 - base);
            __syncthreads();
            if ((int)threadIdx.x < n) {
                const int id = all ? base + threadIdx.x : J.tlist[base + threadIdx.x];
                sid[threadIdx.x] = id;
                sr[threadIdx.x] = J.rec[id];
            }
            __syncthreads();
            for (int k = 0; k < n; ++k) rt_pixel(sr[k], sid[k], x, y, zb, tb);
        }
        if (nchunks == 1) {
            rt_write(J, cam, x, y, zb, tb);
        } else {
            J.pz[(size_t)item * 256 + threadIdx.x] = zb;
            J.pid[(size_t)item * 256 + threadIdx.x] = tb;
        }
    }
}

// lexicographic (depth, id) minimum over the chunks of multi-chunk tiles
__global__ void __launch_bounds__(256) k_rt_merge(JobArg<RasterJob> jobs, CamDev cam, int ntx, int nt) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    if (J.ioff[nt] == nt) return;   // one item per tile: no tile was split, nothing to merge
    for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
        const int i0 = J.ioff[tile], i1 = J.ioff[tile + 1];
        if (i1 - i0 <= 1) continue;
        unsigned long long zb = 0x7ff0000000000000ULL;
        int tb = INT_MAX;
        for (int i = i0; i < i1; ++i) {
            const unsigned long long z = J.pz[(size_t)i * 256 + threadIdx.x];
            const int id = J.pid[(size_t)i * 256 + threadIdx.x];
            if (z < zb || (z == zb && id < tb)) { zb = z; tb = id; }
        }
        const int x = (tile % ntx) * LC_RT_TILE + (threadIdx.x & (LC_RT_TILE - 1));
        const int y = (tile / ntx) * LC_RT_TILE + (threadIdx.x >> LC_RT_SHIFT);
        rt_write(J, cam, x, y, zb, tb);
    }
}


// attributes / ids of the winning triangle (mode 1 / 2, rasterizer.py:58-68)
__device__ __forceinline__ int id_pick(double l0, double l1, double l2) {
    if (l0 >= l1 && l0 >= l2) return 0;
    if (l1 >= l2) return 1;
    return 2;
}

__global__ void k_raster_resolve(JobArg<RasterJob> jobs, CamDev cam, const int *tris, int mode,
                                 const double *attrs, int n_attr, const int *ids, double bg_attr,
                                 long long bg_id, double *zout, double *aout, long long *iout) {
    lc_pdl_wait();
    const RasterJob J = jobs[blockIdx.y];
    const int HW = cam.W * cam.H;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) {
        zout[i] = __longlong_as_double((long long)J.zbuf[i]);
        const int t = J.tri_id[i];
        if (mode == 0) continue;
        if (t == INT_MAX) {
            if (mode == 1)
                for (int k = 0; k < n_attr; ++k) aout[(size_t)i * n_attr + k] = bg_attr;
            else
                iout[i] = bg_id;
            continue;
        }
        double P[3][2], D[3], inv;
        int bb[4];
        tri_setup(cam, J.verts, tris, t, P, D, inv, bb);
        double l0, l1, l2;
        bary(P, inv, i % cam.W, i / cam.W, l0, l1, l2);
        const int v0 = tris[3 * t], v1 = tris[3 * t + 1], v2 = tris[3 * t + 2];
        if (mode == 1) {
            for (int k = 0; k < n_attr; ++k)
                aout[(size_t)i * n_attr + k] = l0 * attrs[(size_t)v0 * n_attr + k]
                                             + l1 * attrs[(size_t)v1 * n_attr + k]
                                             + l2 * attrs[(size_t)v2 * n_attr + k];
        } else {
            const int w = id_pick(l0, l1, l2);
            iout[i] = ids[w == 0 ? v0 : (w == 1 ? v1 : v2)];
        }
    }
}

// ===========================================================================
// kinematics / skinning

__global__ void k_fk(JobArg<FkJob> jobs, const SkelDev *sk) {
    lc_pdl_wait();
    const FkJob J = jobs[blockIdx.x];
    if (!J.active) return;
    __shared__ FkState f;
    fk_warp(*sk, J.x, f);
    // copy out (plain struct of doubles/ints)
    const double *src = reinterpret_cast<const double *>(&f);
    double *dst = reinterpret_cast<double *>(J.fk);
    const int nd = (int)(sizeof(FkState) / sizeof(double));
    for (int i = threadIdx.x; i < nd; i += blockDim.x) dst[i] = src[i];
}

struct GlobalDq {
    const FkState *f;
    __device__ __forceinline__ double operator()(int j, int k) const { return f->dq[j][k]; }
};

__global__ void k_skin(JobArg<SkinJob> jobs, ActorDev A) {
    lc_pdl_wait();
    const SkinJob J = jobs[blockIdx.y];
    if (!J.active) return;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= J.M) return;
    const int v = J.subset ? J.subset[m] : m;
    V3 r = ld3(J.rest + 3 * (size_t)m);
    if (J.disp) r = r + ld3(J.disp + 3 * (size_t)m);
    Blend B;
    dq_blend(A.skin_idx + 4 * v, A.skin_w + 4 * v, A.dominant[v], GlobalDq{J.fk}, B);
    Q4 cr;
    const V3 p = dq_apply(B, r, cr);
    st3(J.pos + 3 * (size_t)m, p);
    if (J.rot) {
        double *q = J.rot + 4 * (size_t)m;
        q[0] = cr.w; q[1] = cr.x; q[2] = cr.y; q[3] = cr.z;
    }
}

// ===========================================================================
// occluding contour vertices (extract_contour_vertices, pose_stage.py:151-191)

__global__ void k_tri_front(JobArg<ContourJob> jobs, ActorDev A) {
    lc_pdl_wait();
    const ContourJob J = jobs[blockIdx.y];
    if (!J.active) return;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < A.T; t += gridDim.x * blockDim.x) {
        const V3 p0 = ld3(J.verts + 3 * (size_t)A.tris[3 * t]);
        const V3 p1 = ld3(J.verts + 3 * (size_t)A.tris[3 * t + 1]);
        const V3 p2 = ld3(J.verts + 3 * (size_t)A.tris[3 * t + 2]);
        const V3 n = cross3(p1 - p0, p2 - p0);
        const V3 c = v3(((p0.x + p1.x) + p2.x) / 3.0, ((p0.y + p1.y) + p2.y) / 3.0,
                        ((p0.z + p1.z) + p2.z) / 3.0);
        J.tri_front[t] = dot3(n, c) < 0.0;
        st3(J.tri_n + 3 * (size_t)t, n);
    }
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < A.N; v += gridDim.x * blockDim.x)
        J.vflag[v] = 0;
}

__global__ void k_sil_edges(JobArg<ContourJob> jobs, ActorDev A) {
    lc_pdl_wait();
    const ContourJob J = jobs[blockIdx.y];
    if (!J.active) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.E; e += gridDim.x * blockDim.x) {
        const int ta = A.edge_tris[2 * e], tb = A.edge_tris[2 * e + 1];
        const bool sil = tb < 0 ? J.tri_front[ta] != 0 : (J.tri_front[ta] != J.tri_front[tb]);
        if (sil) {
            J.vflag[A.edges[2 * e]] = 1;
            J.vflag[A.edges[2 * e + 1]] = 1;
        }
    }
}

// z <= zbuf[rint(pix)] + 0.01 z  with in-image test (pose_stage.py:175-181,
// nonrigid_stage.py:93-99)
__device__ __forceinline__ bool depth_visible(CamDev cam, const unsigned long long *zbuf, V3 p) {
    double px, py;
    const bool ok = project(cam, p, px, py);
    const double xr = fmin(fmax(rint(px), 0.0), (double)(cam.W - 1));
    const double yr = fmin(fmax(rint(py), 0.0), (double)(cam.H - 1));
    const bool inimg = px >= -0.5 && px <= cam.W - 0.5 && py >= -0.5 && py <= cam.H - 0.5;
    const double zb = __longlong_as_double((long long)zbuf[(size_t)yr * cam.W + (size_t)xr]);
    return ok && inimg && (p.z <= zb + 0.01 * p.z);
}

// one CTA per stream: ordered compaction of contour candidates (np.unique
// order = ascending vertex id) and, optionally, of visible vertices; then the
// image-plane normals of the contour vertices.
// the depth-visibility test of every vertex, grid-wide (the compaction below
// is one CTA per stream and only scans these flags): vflag[v] becomes
// bit 0 = visible, bit 1 = visible and on a silhouette edge
__global__ void k_vis_flags(JobArg<ContourJob> jobs, ActorDev A, CamDev cam) {
    lc_pdl_wait();
    const ContourJob J = jobs[blockIdx.y];
    if (!J.active) return;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < A.N; v += gridDim.x * blockDim.x) {
        const bool vis = depth_visible(cam, J.zbuf, ld3(J.verts + 3 * (size_t)v));
        J.vflag[v] = (uint8_t)((vis ? 1 : 0) | ((vis && J.vflag[v]) ? 2 : 0));
    }
}

__global__ void __launch_bounds__(1024) k_contour_compact(JobArg<ContourJob> jobs, ActorDev A,
                                                          CamDev cam) {
    lc_pdl_wait();
    const ContourJob J = jobs[blockIdx.x];
    if (!J.active) return;
    // each thread owns a run of consecutive vertices: count both lists' flags,
    // one block scan of the (contour, visible) count pairs, then every
    // thread writes its run in ascending order (two block barriers in all)
    __shared__ unsigned long long wsum[32];
    __shared__ int tot[2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int per = (A.N + blockDim.x - 1) / blockDim.x;
    const int v0 = min(A.N, (int)threadIdx.x * per), v1 = min(A.N, v0 + per);
    unsigned long long cnt = 0;   // contour count | visible count << 32
    for (int v = v0; v < v1; ++v) {
        const int fl = J.vflag[v];   // (k_vis_flags)
        cnt += ((fl & 2) ? 1ull : 0ull) + ((fl & 1) ? (1ull << 32) : 0ull);
    }
    unsigned long long inc = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long u = lane < nw ? wsum[lane] : 0ull;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, u, o);
            if (lane >= o) u += t;
        }
        if (lane < nw) wsum[lane] = u;   // inclusive warp totals
        if (lane == nw - 1) { tot[0] = (int)(u & 0xffffffffu); tot[1] = (int)(u >> 32); }
    }
    __syncthreads();
    const unsigned long long before = (w > 0 ? wsum[w - 1] : 0ull) + inc - cnt;
    int p0 = (int)(before & 0xffffffffu), p1 = (int)(before >> 32);
    for (int v = v0; v < v1; ++v) {
        const int fl = J.vflag[v];
        if (fl & 2) J.idx[p0++] = v;
        if ((fl & 1) && J.vis) J.vis[p1++] = v;
    }
    __syncthreads();   // the contour ids, for the normals below
    const int B = tot[0];
    if (threadIdx.x == 0) {
        *J.B = B;
        if (J.P) *J.P = J.vis ? tot[1] : 0;
    }
    // vertex normals: area-weighted, accumulated in np.add.at slot order
    // (pose_stage.py:139-148), projected with d(pix)/d(p), normalized
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        const int v = J.idx[b];
        V3 n = v3(0, 0, 0);
        for (int k = A.vt_ptr[v]; k < A.vt_ptr[v + 1]; ++k) n = n + ld3(J.tri_n + 3 * (size_t)A.vt_tri[k]);
        double nn = norm3(n);
        if (nn < 1e-12) nn = 1.0;
        n = v3(n.x / nn, n.y / nn, n.z / nn);
        double a0, a2, b1, b2;
        proj_jac(cam, ld3(J.verts + 3 * (size_t)v), a0, a2, b1, b2);
        double u = a0 * n.x + 0.0 * n.y + a2 * n.z;
        double q = 0.0 * n.x + b1 * n.y + b2 * n.z;
        const double l = sqrt(u * u + q * q);
        if (l > 1e-12) { u = u / l; q = q / l; } else { u = 0.0; q = 0.0; }
        J.n2d[2 * b] = u;
        J.n2d[2 * b + 1] = q;
    }
}

// ===========================================================================
// outer-rim filter (outer_rim_mask, pose_stage.py:218-264) and, for Stage II,
// the body-part gate (pipeline.py:241-249 with build_body_part_mask,
// nonrigid_stage.py:102-128).  One warp per contour vertex.

#define LC_MAX_PARTS 16

// part id of the max-barycentric vertex of the winning triangle at (x, y); 0 = background
__device__ __forceinline__ int part_at(const ActorDev &A, CamDev cam, const double *verts,
                                       const int *tri_id, int x, int y) {
    const int t = tri_id[(size_t)y * cam.W + x];
    if (t == INT_MAX) return 0;
    double P[3][2], D[3], inv;
    int bb[4];
    tri_setup(cam, verts, A.tris, t, P, D, inv, bb);
    double l0, l1, l2;
    bary(P, inv, x, y, l0, l1, l2);
    const int w = id_pick(l0, l1, l2);
    return A.vpart[A.tris[3 * t + w]];
}

// One warp per 16x16 cell (8 cells per CTA): the cell's contour pixels of
// the own mask (foreground with a background 4-neighbour, the image border
// counting as background; imageproc.py:34-49), compacted in row-major order
// two cell rows per ballot (lanes 0-15 the upper row, 16-31 the lower).
__global__ void __launch_bounds__(256) k_own_cells(JobArg<OwnCellsJob> jobs, int H, int W, int ncx) {
    lc_pdl_wait();
    const OwnCellsJob J = jobs[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int ncells = ncx * ((H + LC_GRID_CELL - 1) / LC_GRID_CELL);
    static_assert(LC_GRID_CELL == 16, "two cell rows per warp ballot");
    for (int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < ncells; c += gridDim.x * (blockDim.x >> 5)) {
        const int x = (c % ncx) * LC_GRID_CELL + (lane & 15);
        int n = 0;
        for (int r = 0; r < LC_GRID_CELL; r += 2) {
            const int y = (c / ncx) * LC_GRID_CELL + r + (lane >> 4);
            bool on = false;
            if (x < W && y < H && J.mask[(size_t)y * W + x]) {
                const bool l = x > 0 && J.mask[(size_t)y * W + x - 1], rr = x + 1 < W && J.mask[(size_t)y * W + x + 1];
                const bool u = y > 0 && J.mask[(size_t)(y - 1) * W + x], d = y + 1 < H && J.mask[(size_t)(y + 1) * W + x];
                on = !(l && rr && u && d);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, on);
            if (on) J.keys[(size_t)c * 256 + n + __popc(bal & ((1u << lane) - 1u))] = (y << 16) | x;
            n += __popc(bal);
        }
        if (lane == 0) J.cnt[c] = n;
    }
}

// Is some own-contour pixel at squared distance < lim2 (<= lim2 when
// `inclusive`) from (qx, qy)?  The cells within R >= sqrt(lim2) are scanned
// and the scan stops at the first such pixel.  The squared distance is the
// same expression as the nearest-distance search, so every threshold decision
// on the minimum is reproduced exactly.
__device__ inline bool own_any_within(const NnGridDev &g, const int *cnt, const int *keys, double qx, double qy,
                                      double R, double lim2, bool inclusive) {
    if (!(isfinite(qx) && isfinite(qy))) return false;
    const int cx0 = max(0, (int)floor((qx - R) / LC_GRID_CELL));
    const int cx1 = min(g.ncx - 1, (int)floor((qx + R) / LC_GRID_CELL));
    const int cy0 = max(0, (int)floor((qy - R) / LC_GRID_CELL));
    const int cy1 = min(g.ncy - 1, (int)floor((qy + R) / LC_GRID_CELL));
    for (int cy = cy0; cy <= cy1; ++cy)
        for (int cx = cx0; cx <= cx1; ++cx) {
            const int c = cy * g.ncx + cx;
            const int n = cnt[c];
            const int *kk = keys + (size_t)c * 256;
            for (int k = 0; k < n; ++k) {
                const int key = kk[k];
                const double dx = qx - (double)(key & 0xffff), dy = qy - (double)(key >> 16);
                const double d2 = dx * dx + dy * dy;
                if (inclusive ? d2 <= lim2 : d2 < lim2) return true;
            }
        }
    return false;
}

// own_any_within by a whole warp for one query point (warp-uniform
// arguments): the lanes split each cell's pixels, one vote per cell.
__device__ inline bool own_any_within_warp(const NnGridDev &g, const int *cnt, const int *keys, double qx, double qy,
                                           double R, double lim2, bool inclusive) {
    if (!(isfinite(qx) && isfinite(qy))) return false;
    const int lane = threadIdx.x & 31;
    const int cx0 = max(0, (int)floor((qx - R) / LC_GRID_CELL));
    const int cx1 = min(g.ncx - 1, (int)floor((qx + R) / LC_GRID_CELL));
    const int cy0 = max(0, (int)floor((qy - R) / LC_GRID_CELL));
    const int cy1 = min(g.ncy - 1, (int)floor((qy + R) / LC_GRID_CELL));
    for (int cy = cy0; cy <= cy1; ++cy)
        for (int cx = cx0; cx <= cx1; ++cx) {
            const int c = cy * g.ncx + cx;
            const int n = cnt[c];
            const int *kk = keys + (size_t)c * 256;
            bool hit = false;
            for (int k0 = 0; k0 < n; k0 += 32) {
                const int k = k0 + lane;
                if (k < n) {
                    const int key = kk[k];
                    const double dx = qx - (double)(key & 0xffff), dy = qy - (double)(key >> 16);
                    const double d2 = dx * dx + dy * dy;
                    hit = hit || (inclusive ? d2 <= lim2 : d2 < lim2);
                }
            }
            if (__any_sync(0xffffffffu, hit)) return true;
        }
    return false;
}

#define LC_RIM_LIST 128   // own-contour pixels near one rim vertex, per warp
__global__ void __launch_bounds__(256) k_rim(JobArg<RimJob> jobs, ActorDev A, CamDev cam, const double *probe_offs) {
    lc_pdl_wait();
    const RimJob J = jobs[blockIdx.y];
    if (!J.active) return;
    const int B = *J.B;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const NnGridDev own = J.own;
    __shared__ int near_all[8][LC_RIM_LIST];   // one list per warp: launched with 256 threads
    int *near = near_all[threadIdx.x >> 5];
    for (int b = blockIdx.x * wpb + (threadIdx.x >> 5); b < B; b += gridDim.x * wpb) {
        const int v = J.idx[b];
        const V3 p = ld3(J.verts + 3 * (size_t)v);
        double px, py;
        const bool ok = project(cam, p, px, py);
        // outer_rim_mask (pose_stage.py:218-264): keep iff the own-mask
        // contour is within 1.5 px, and in Stage I some interior probe is at
        // least 6 px (2 * depth >= 12) from it.  Both are threshold tests, so
        // bounded exact searches decide them (nn_within2).
        // sqrt is correctly rounded and monotone with sqrt(2.25) = 1.5 and
        // sqrt(36) = 6 exact, so sqrt(d2) <= 1.5 <=> d2 <= 2.25 and
        // sqrt(d2) >= 6 <=> d2 >= 36: the threshold tests on the nearest
        // distance become "is any contour pixel that close" (early exit)
        bool keep = false;
        if (ok) keep = own_any_within_warp(own, J.own_cnt, J.own_keys, px, py, 2.0, 2.25, true);
        if (J.stage1) {
            if (keep) {
                // 16 directions x radii 1..8: depth = max over interior probes
                // of the nearest contour distance, keep iff 2 * depth >= 12,
                // i.e. iff some interior probe has no contour pixel closer
                // than 6 px; lane = (direction, half of the radii).  A pixel
                // within 6 px of a probe (at most 8 px out) is within 14 px of
                // the vertex: the warp first gathers the pixels within 15 px
                // (d2 <= 226, a superset through any rounding) into shared
                // memory, and every probe scans that short list (broadcast
                // reads); a list over LC_RIM_LIST falls back to the cell scans
                int nl = 0;
                {
                    const double R = 15.0;
                    const int cx0 = max(0, (int)floor((px - R) / LC_GRID_CELL));
                    const int cx1 = min(own.ncx - 1, (int)floor((px + R) / LC_GRID_CELL));
                    const int cy0 = max(0, (int)floor((py - R) / LC_GRID_CELL));
                    const int cy1 = min(own.ncy - 1, (int)floor((py + R) / LC_GRID_CELL));
                    for (int cy = cy0; cy <= cy1; ++cy)
                        for (int cx = cx0; cx <= cx1; ++cx) {
                            const int c = cy * own.ncx + cx;
                            const int n = J.own_cnt[c];
                            const int *kk = J.own_keys + (size_t)c * 256;
                            for (int k0 = 0; k0 < n; k0 += 32) {
                                const int k = k0 + lane;
                                bool take = false;
                                int key = 0;
                                if (k < n) {
                                    key = kk[k];
                                    const double dx = px - (double)(key & 0xffff), dy = py - (double)(key >> 16);
                                    take = dx * dx + dy * dy <= 226.0;
                                }
                                const unsigned bal = __ballot_sync(0xffffffffu, take);
                                const int at = nl + __popc(bal & ((1u << lane) - 1u));
                                if (take && at < LC_RIM_LIST) near[at] = key;
                                nl += __popc(bal);
                            }
                        }
                    __syncwarp();
                }
                const bool listed = nl <= LC_RIM_LIST;
                bool deep = false;
                const int dir = lane >> 1, r0 = (lane & 1) * 4;
                for (int r = r0; r < r0 + 4; ++r) {
                    const int k = dir * 8 + r;
                    const double qx = px + probe_offs[2 * k], qy = py + probe_offs[2 * k + 1];
                    if (field_inside(own, qx, qy)) {
                        bool shallow = false;
                        if (listed) {
                            for (int j = 0; j < nl && !shallow; ++j) {
                                const int key = near[j];
                                const double dx = qx - (double)(key & 0xffff), dy = qy - (double)(key >> 16);
                                shallow = dx * dx + dy * dy < 36.0;
                            }
                        } else {
                            shallow = own_any_within(own, J.own_cnt, J.own_keys, qx, qy, 6.0, 36.0, false);
                        }
                        if (!shallow) deep = true;
                    }
                    if (__any_sync(0xffffffffu, deep)) break;   // warp-uniform
                }
                keep = __any_sync(0xffffffffu, deep);
                __syncwarp();   // the list is rewritten for the warp's next vertex
            }
            keep = keep && A.rigidity[v] >= 2.0;
        } else if (J.part_gate) {
            // label image value at rint(pix) clipped into the image
            const int xi = (int)fmin(fmax(rint(px), 0.0), (double)(cam.W - 1));
            const int yi = (int)fmin(fmax(rint(py), 0.0), (double)(cam.H - 1));
            int label = part_at(A, cam, J.verts, J.tri_id, xi, yi);
            if (label == 0) {
                // bounded dilation: nearest part pixel per part within `dilation`
                const int R = J.dilation;
                int best[LC_MAX_PARTS];
                for (int q = 0; q < LC_MAX_PARTS; ++q) best[q] = INT_MAX;
                const int side = 2 * R + 1;
                for (int k = lane; k < side * side; k += 32) {
                    const int dx = k % side - R, dy = k / side - R;
                    const int x = xi + dx, y = yi + dy;
                    if (x < 0 || y < 0 || x >= cam.W || y >= cam.H) continue;
                    const int d2 = dx * dx + dy * dy;
                    if (d2 > R * R) continue;
                    const int pp = part_at(A, cam, J.verts, J.tri_id, x, y);
                    if (pp > 0 && pp < LC_MAX_PARTS && d2 < best[pp]) best[pp] = d2;
                }
                for (int q = 1; q < LC_MAX_PARTS; ++q)
                    for (int o = 16; o > 0; o >>= 1)
                        best[q] = min(best[q], __shfl_xor_sync(0xffffffffu, best[q], o));
                int arg = 0, bd = INT_MAX;
                for (int q = 1; q < LC_MAX_PARTS; ++q)
                    if (best[q] < bd) { bd = best[q]; arg = q; }   // lowest id on ties
                label = arg;
                if (best[1] != INT_MAX) label = 1;                // torso override (TORSO_PART = 1)
            }
            keep = keep && ok && (label == 0 || label == A.vpart[v]);
        }
        if (lane == 0) J.keep[b] = keep;
    }
}

// Full body-part label image (build_body_part_mask, nonrigid_stage.py:102-128)
// for the set-parity seam: the label k_rim reads at one pixel, evaluated at
// every pixel with the same device logic (own part from the winning
// triangle's max-barycentric vertex; background pixels take the nearest part
// within `dilation` px, lowest id on ties, torso override).
__global__ void k_part_labels(ActorDev A, CamDev cam, const double *verts, const int *tri_id, int dilation,
                              int *labels) {
    lc_pdl_wait();
    const long long HW = (long long)cam.W * cam.H;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < HW; q += (long long)gridDim.x * blockDim.x) {
        const int xi = (int)(q % cam.W), yi = (int)(q / cam.W);
        int label = part_at(A, cam, verts, tri_id, xi, yi);
        if (label == 0) {
            const int R = dilation;
            int best[LC_MAX_PARTS];
            for (int k = 0; k < LC_MAX_PARTS; ++k) best[k] = INT_MAX;
            for (int dy = -R; dy <= R; ++dy)
                for (int dx = -R; dx <= R; ++dx) {
                    const int x = xi + dx, y = yi + dy;
                    if (x < 0 || y < 0 || x >= cam.W || y >= cam.H) continue;
                    const int d2 = dx * dx + dy * dy;
                    if (d2 > R * R) continue;
                    const int pp = part_at(A, cam, verts, tri_id, x, y);
                    if (pp > 0 && pp < LC_MAX_PARTS && d2 < best[pp]) best[pp] = d2;
                }
            int arg = 0, bd = INT_MAX;
            for (int k = 1; k < LC_MAX_PARTS; ++k)
                if (best[k] < bd) { bd = best[k]; arg = k; }
            label = arg;
            if (best[1] != INT_MAX) label = 1;
        }
        labels[q] = label;
    }
}

// (M,3,36) skinning Jacobian for the lc_skin_points seam (skin_points with
// dq_jacobian, skinning.py:391-397); the per-joint DQ Jacobian columns are
// recomputed from the FK state on the fly.
__global__ void k_skin_jac(const FkState *fk, const SkelDev *skg, ActorDev A, int M, const double *rest,
                           const int *subset, double *jac) {
    lc_pdl_wait();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    const SkelDev &sk = *skg;
    const int v = subset ? subset[m] : m;
    const V3 r = ld3(rest + 3 * (size_t)m);
    Blend B;
    dq_blend(A.skin_idx + 4 * v, A.skin_w + 4 * v, A.dominant[v], GlobalDq{fk}, B);
    double dv[3][8];
    dq_dtransform(B, r, dv);
    for (int q = 0; q < LC_NP; ++q) {
        double db[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int nsl = B.degenerate ? 1 : 4;
        for (int sl = 0; sl < nsl; ++sl) {
            const int j = B.degenerate ? B.dom : B.js[sl];
            const double cf = B.degenerate ? 1.0 : B.coef[sl];
            double col[8];
            if (q >= 3 && q < 6) {
                const Q4 d = dq_trans(*fk, j, q - 3);
                col[0] = col[1] = col[2] = col[3] = 0.0;
                col[4] = d.w; col[5] = d.x; col[6] = d.y; col[7] = d.z;
            } else if (q >= 33) {
                for (int k = 0; k < 8; ++k) col[k] = 0.0;
            } else {
                dq_spin(sk, *fk, j, q < 3 ? q : q - 3, col);
            }
            for (int k = 0; k < 8; ++k) db[k] += cf * col[k];
        }
        for (int i = 0; i < 3; ++i) {
            double a = 0.0;
            for (int k = 0; k < 8; ++k) a += dv[i][k] * db[k];
            jac[((size_t)m * 3 + i) * LC_NP + q] = a;
        }
    }
}
