// lattice.cu -- the near field of translation-invariant leaves as dense
// GEMMs on the FP64 tensor cores.
//
// The paper's discretisation covers the interior with a regular lattice of
// boxes that all carry the same node set; when the reference tree's leaves
// line up with that lattice (cfg4: 2 x 2 boxes, 256 nodes per leaf), every
// leaf holds a translate of one point pattern, and the near-field block
// between a leaf and its neighbour at offset o = (dx, dy),
//     K_o[i][j] = ln |r_i - r_j - o pitch|^2      (0 where r^2 == 0:
//                                                  summation.cpp:340),
// is the SAME matrix for every leaf.  The geometry is static, so the nine
// K_o (m x m each) are formed once per plan, and an apply's near field,
// summation.cpp:330-344 for all leaves at once, is
//     N[:, A] = sum_o K_o . q[:, A + o]           (m x nleaf),
// a real dense contraction with 2 flop per pair instead of a log per pair:
// it goes to the tensor cores (mma.sync m8n8k4 f64), like M2L.  The plan
// takes this path only when it verified the congruence on the actual
// coordinates: every non-empty leaf has the pattern's point count and every
// point sits within a few ulp of pattern + leaf translation; anything else
// keeps the pairwise kernels (fmm.cu, sym.cuh).
//
// Kernel: a CTA owns NT leaves (columns) and all m rows; it walks the 9 x
// m/32 k-chunks.  The A chunk (K_o[:, 32 k], 66 KB with the conflict-free
// leading dimension m + 4, contiguous in global memory) arrives by 1-D TMA
// bulk copies on an mbarrier, double-buffered; the B chunk (32 charges of
// each of the NT neighbour leaves, contiguous runs of the Morton-sorted
// charge vector, zeros outside the domain) is prefetched into registers one
// chunk ahead.  Warp w owns row tiles w MTW .. w MTW + MTW - 1 and all
// column tiles; accumulators stay in registers for the whole k range; the
// sums go to the one-slot partial array that sym_finalize_kernel (fmm.cu)
// turns into potentials together with the far field.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "plan.cuh"

namespace vpg {
namespace {

#ifndef VPG_LAT_UNROLL
#define VPG_LAT_UNROLL 8
#endif
constexpr int kLatUnroll = VPG_LAT_UNROLL;  // k-steps unrolled
constexpr int kLatKC = 32;        // k per chunk
constexpr int kLatThreads = 256;  // 8 warps
constexpr int kLatLB = kLatKC + 4;

__host__ __device__ constexpr int lat_la(int m) { return m + 4; }  // == 4 mod 16 for m % 16 == 0

// K_o[i][j] in the kernel's chunk order: [o][kc][kk][la], element (kk, i) = K_o[i][32 kc + kk]
__global__ void lat_build_kernel(const double2* pat, int m, double px, double py, double* K) {
    const int la = lat_la(m);
    const int64_t total = int64_t(9) * m * la;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % la);
        const int64_t r = e / la;
        const int j = int(r % m), o = int(r / m);
        double v = 0.0;
        if (i < m) {
            const int dx = o % 3 - 1, dy = o / 3 - 1;
            const double2 a = pat[i], b = pat[j];
            const double ddx = a.x - (b.x + dx * px), ddy = a.y - (b.y + dy * py);
            const double r2 = fma(ddy, ddy, ddx * ddx);
            v = r2 == 0.0 ? 0.0 : log(r2);
        }
        K[e] = v;  // e == ((o * m + j) * la + i): chunks of 32 consecutive j are contiguous
    }
}

__device__ __forceinline__ void lat_dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// KB: k extent of a block (the pattern's point count), NBLK: blocks per column (9 neighbour leaves
// for the near field; 1 for the pattern's power sums, lattice_p2m_issue)
template <int MTW, int NT, int KB, int NBLK>
__global__ void __launch_bounds__(kLatThreads, 1)
lattice_near_kernel(const double* K, const int32_t* nbr, const double* qs, int ncol, double* near) {
    constexpr int m = 64 * MTW, la = lat_la(m), kNt = NT / 8, kChunks = NBLK * (KB / kLatKC);
    constexpr uint32_t kChunkBytes = uint32_t(kLatKC) * la * 8u;
    extern __shared__ __align__(16) double ls[];
    double* As = ls;                                // [2][kLatKC][la]
    double* Bs = ls + 2 * size_t(kLatKC) * la;      // [NT][kLatLB]
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    uint32_t use0 = 0u, use1 = 0u;  // completed phases per buffer (same in every thread)
    const int bj = tid >> 2, bpart = tid & 3;  // B fetch: column bj, doubles 8 bpart .. + 7 of the chunk
    const int ntiles = (ncol + NT - 1) / NT;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int n0 = tile * NT, nc = min(NT, ncol - n0);
        double acc[MTW][kNt][2];
#pragma unroll
        for (int i = 0; i < MTW; ++i)
#pragma unroll
            for (int t = 0; t < kNt; ++t) acc[i][t][0] = acc[i][t][1] = 0.0;
        double2 breg[4];
        auto issue_a = [&](int c) {
            if (tid == 0) {
                uint64_t* b = &bar[c & 1];
                mbar_arrive_expect_tx(b, kChunkBytes);
                const char* src = reinterpret_cast<const char*>(K) + size_t(c) * kChunkBytes;
                char* dst = reinterpret_cast<char*>(As + size_t(c & 1) * kLatKC * la);
                for (uint32_t off = 0; off < kChunkBytes; off += 32768u)
                    tma_load_1d(dst + off, src + off, min(32768u, kChunkBytes - off), b);
            }
        };
        auto fetch_b = [&](int c) {
            const int o = c / (KB / kLatKC), kc = c % (KB / kLatKC);
#pragma unroll
            for (int r = 0; r < 4; ++r) breg[r] = make_double2(0.0, 0.0);
            if (bj < nc) {
                const int src = nbr[int64_t(n0 + bj) * NBLK + o];
                if (src >= 0) {
                    const double2* p = reinterpret_cast<const double2*>(qs + src + kc * kLatKC + bpart * 8);
#pragma unroll
                    for (int r = 0; r < 4; ++r) breg[r] = p[r];
                }
            }
        };
        __syncthreads();  // the previous tile's reads of As / Bs are done
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_a(0);
        fetch_b(0);
        for (int c = 0; c < kChunks; ++c) {
            __syncthreads();  // chunk c - 1 consumed: Bs and the other A buffer are free
            if (bj < NT) {
                double2* d = reinterpret_cast<double2*>(Bs + bj * kLatLB + bpart * 8);
#pragma unroll
                for (int r = 0; r < 4; ++r) d[r] = breg[r];
            }
            if (c + 1 < kChunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_a(c + 1);
                fetch_b(c + 1);
            }
            if (c & 1) mbar_wait(&bar[1], use1++ & 1u);
            else mbar_wait(&bar[0], use0++ & 1u);
            __syncthreads();  // Bs written
            const double* Ab = As + size_t(c & 1) * kLatKC * la;
#pragma unroll(kLatUnroll)
            for (int k4 = 0; k4 < kLatKC; k4 += 4) {
                double a[MTW], b[kNt];
#pragma unroll
                for (int i = 0; i < MTW; ++i) a[i] = Ab[(k4 + kq) * la + 8 * (warp * MTW + i) + rq];
#pragma unroll
                for (int t = 0; t < kNt; ++t) b[t] = Bs[(8 * t + rq) * kLatLB + k4 + kq];
#pragma unroll
                for (int i = 0; i < MTW; ++i)
#pragma unroll
                    for (int t = 0; t < kNt; ++t) lat_dmma(acc[i][t][0], acc[i][t][1], a[i], b[t]);
            }
        }
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
            const int row = 8 * (warp * MTW + i) + rq;
#pragma unroll
            for (int t = 0; t < kNt; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = 8 * t + 2 * kq + h;
                    if (col < nc) near[int64_t(n0 + col) * m + row] = acc[i][t][h];
                }
        }
    }
}

template <int MTW, int NT>
size_t lat_smem() {  // (independent of KB / NBLK)
    constexpr int m = 64 * MTW;
    return sizeof(double) * (2 * size_t(kLatKC) * lat_la(m) + size_t(NT) * kLatLB);
}

template <int MTW, int NT>
void lat_launch(const Plan& pl, const double* qs, double* near, cudaStream_t st) {
    const size_t smem = lat_smem<MTW, NT>();
    smem_optin((const void*)lattice_near_kernel<MTW, NT, 64 * MTW, 9>, int(smem));
    const int ntiles = int((pl.lat_ncol + NT - 1) / NT);
    launch_pdl(lattice_near_kernel<MTW, NT, 64 * MTW, 9>, dim3(unsigned(std::min(ntiles, pl.sm_count))),
               dim3(kLatThreads), smem, st, (const double*)pl.lat_K.p, (const int32_t*)pl.lat_nbr.p, qs,
               int(pl.lat_ncol), near);
}

template <int MTW>
void lat_launch_nt(const Plan& pl, const double* qs, double* near, cudaStream_t st) {
    switch (pl.lat_nt) {
        case 40: return lat_launch<MTW, 40>(pl, qs, near, st);
        case 48: return lat_launch<MTW, 48>(pl, qs, near, st);
        case 56: return lat_launch<MTW, 56>(pl, qs, near, st);
        default: return lat_launch<MTW, 64>(pl, qs, near, st);
    }
}


// ---- P2M of lattice plans.  Every leaf is the pattern shifted by its translation, and the
// tree's box centres drift against the lattice by d_A = (translation - centre offset) / s
// (the bounding box is not a multiple of the pitch: |d| <= ~2% of a box on cfg4), so with
// w0_j the pattern's points about the pattern leaf's centre,
//   sum_j q_j (w0_j + d_A)^k = sum_{i <= k} C(k, i) d_A^(k - i) S_i(A),   S_i(A) = sum_j q_j w0_j^i:
// the power sums S (re, im rows of the fixed matrix V = w0^i, 2 (P + 1) <= 128 rows) are ONE
// GEMM V . q for all leaves on the tensor cores (the kernel above, one block per column), and a
// warp per leaf applies the binomial shift and the -1/k (summation.cpp:247-254's multipoles
// to rounding; the coordinates enter through the pattern as in the near field).
constexpr int kLatSRows = 128;

__global__ void __launch_bounds__(128)
lat_p2m_shift_kernel(const double* S, const double2* drift, const int32_t* rows, const double* binom, int ncol,
                     int P, int J, double2* mult) {
    __shared__ double2 sp[4][64], dp[4][64];
    __shared__ double bsm[51 * 51];  // C(k, i): lanes differ in k, so not the constant bank
    for (int i = threadIdx.x; i < 51 * 51; i += blockDim.x) bsm[i] = binom[i];
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = P + 1;
    for (int col = blockIdx.x * 4 + warp; col < ncol; col += gridDim.x * 4) {
        const double2 d = drift[col];
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = lane + 32 * h;
            if (i <= P) {
                sp[warp][i] = make_double2(S[int64_t(col) * kLatSRows + 2 * i], S[int64_t(col) * kLatSRows + 2 * i + 1]);
                double2 r = make_double2(1.0, 0.0), b = d;  // d^i by binary powering
                for (int e = i; e; e >>= 1) {
                    if (e & 1) r = make_double2(r.x * b.x - r.y * b.y, r.x * b.y + r.y * b.x);
                    b = make_double2(b.x * b.x - b.y * b.y, 2.0 * b.x * b.y);
                }
                dp[warp][i] = r;
            }
        }
        __syncwarp();
        double2* dst = mult + int64_t(rows[col]) * n;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = lane + 32 * h;
            const int kk = min(k, P);             // idle lanes shadow k = P (result dropped)
            const int kmax = min(31 + 32 * h, P);  // the warp's longest sum: one trip count for every lane
            const double* brow = bsm + kk * 51;
            double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;  // two interleaved partial sums (even / odd i)
            // terms with k - i > J are below 1e-17 of the coefficient's scale (J from the plan's
            // largest drift, build_lattice_p2m): the warp starts at its smallest useful i
            const int ilo = max(0, (32 * h - J) & ~1);
            for (int i = ilo; i <= kmax; i += 2) {
                const int j0 = kk - i, j1 = kk - i - 1;
                const double c0 = (i <= kk && j0 <= J) ? brow[i] : 0.0, c1 = (i + 1 <= kk && j1 <= J) ? brow[i + 1] : 0.0;
                const double2 s0 = sp[warp][i], s1 = sp[warp][min(i + 1, P)];
                const double2 t0 = dp[warp][max(j0, 0)], t1 = dp[warp][max(j1, 0)];
                ar = fma(c0, s0.x * t0.x - s0.y * t0.y, ar);
                ai = fma(c0, s0.x * t0.y + s0.y * t0.x, ai);
                br = fma(c1, s1.x * t1.x - s1.y * t1.y, br);
                bi = fma(c1, s1.x * t1.y + s1.y * t1.x, bi);
            }
            if (k <= P) {
                const double f = k ? -1.0 / double(k) : 1.0;
                dst[k] = make_double2(f * (ar + br), k ? f * (ai + bi) : 0.0);
            }
        }
    }
}

template <int NT, int KB>
void lat_p2m_launch(const Plan& pl, const double* qs, double* S, cudaStream_t st) {
    const size_t smem = lat_smem<2, NT>();
    smem_optin((const void*)lattice_near_kernel<2, NT, KB, 1>, int(smem));
    const int ntiles = int((pl.lat_p2m_ncol + NT - 1) / NT);
    launch_pdl(lattice_near_kernel<2, NT, KB, 1>, dim3(unsigned(std::min(ntiles, pl.sm_count))), dim3(kLatThreads),
               smem, st, (const double*)pl.lat_V.p, (const int32_t*)pl.lat_p2m_src.p, qs, int(pl.lat_p2m_ncol), S);
}

}  // namespace

// The apply's near field: near[col m + i] = sum over the 3 x 3 leaves of K_o q.
void lattice_near_issue(const Plan& pl, const double* qs, double* near, cudaStream_t st) {
    switch (pl.lat_m) {
        case 64: return lat_launch_nt<1>(pl, qs, near, st);
        case 128: return lat_launch_nt<2>(pl, qs, near, st);
        default: return lat_launch_nt<4>(pl, qs, near, st);
    }
}

// P2M of a lattice plan: S = V q for every non-empty leaf, then the per-leaf shift into the
// multipole rows.  S: scratch of lat_p2m_ncol x 128 doubles.
void lattice_p2m_issue(const Plan& pl, const double* qs, double* S, double2* mult, cudaStream_t st) {
    switch (pl.lat_m) {
        case 64: lat_p2m_launch<64, 64>(pl, qs, S, st); break;
        case 128: lat_p2m_launch<64, 128>(pl, qs, S, st); break;
        default: lat_p2m_launch<64, 256>(pl, qs, S, st); break;
    }
    const unsigned grid = unsigned(std::min<int64_t>((pl.lat_p2m_ncol + 3) / 4, int64_t(pl.sm_count) * 8));
    launch_pdl(lat_p2m_shift_kernel, dim3(grid), dim3(128), 0, st, (const double*)S, (const double2*)pl.lat_drift.p,
               (const int32_t*)pl.lat_p2m_rows.p, (const double*)pl.lat_binom.p, int(pl.lat_p2m_ncol), pl.P,
               pl.lat_shift_terms, mult);
}

// Host side of the lattice P2M (called by build_lattice_near once the pattern is verified).
static void build_lattice_p2m(Plan& pl, const double2* pat, int64_t first, double px, double py) {
    pl.lat_p2m = false;
    const char* ev = std::getenv("VPG_LATTICE_P2M");
    if (ev && std::atoi(ev) == 0) return;
    const int P = pl.P, L = pl.L, m = pl.lat_m;
    if (P > 50 || 2 * (P + 1) > kLatSRows || pl.up_cap != 0 || pl.multilevel_up || pl.n_p2m_splits > 0) return;
    const int64_t nleaf = int64_t(1) << (2 * L);
    const std::vector<int32_t>& so = pl.h_soff;
    const double s = pl.side / double(1 << L);
    const int fx = int(squash2(uint32_t(first))), fy = int(squash2(uint32_t(first) >> 1));
    const double c0x = pl.x0 + (fx + 0.5) * s, c0y = pl.y0 + (fy + 0.5) * s;
    // V in the kernel's chunk order: [kc][kk][la], element (kk, r) = V[r][32 kc + kk], rows r = 2 i + part
    const int la = lat_la(kLatSRows);
    std::vector<double> V(size_t(m) * la, 0.0);
    for (int j = 0; j < m; ++j) {
        const long double wr = ((long double)pat[j].x - c0x) / s, wi = ((long double)pat[j].y - c0y) / s;
        long double pr = 1.0L, pi = 0.0L;
        for (int i = 0; i <= P; ++i) {
            V[size_t(j) * la + 2 * i] = double(pr);
            V[size_t(j) * la + 2 * i + 1] = double(pi);
            const long double nr = pr * wr - pi * wi;
            pi = pr * wi + pi * wr;
            pr = nr;
        }
    }
    std::vector<int32_t> src, rows;
    std::vector<double2> drift;
    int64_t items = 0;
    for (int64_t b = 0; b < nleaf; ++b) {
        if (so[size_t(b) + 1] == so[size_t(b)]) continue;
        const int ix = int(squash2(uint32_t(b))), iy = int(squash2(uint32_t(b) >> 1));
        src.push_back(so[size_t(b)]);
        rows.push_back(int32_t(lvl_base(L) - lvl_base(2) + b));
        // translation of the leaf's points minus the offset of its box centre, in box units
        const long double tx = (long double)(ix - fx) * px, ty = (long double)(iy - fy) * py;
        const long double cx = (long double)pl.x0 + (ix + 0.5L) * s, cy = (long double)pl.y0 + (iy + 0.5L) * s;
        drift.push_back(make_double2(double((tx - (cx - c0x)) / s), double((ty - (cy - c0y)) / s)));
        ++items;
    }
    if (items != pl.n_p2m_items) return;  // the P2M items are exactly the non-empty leaves
    // shift series cut: C(P, J) (dmax / 0.7)^J < 1e-17 of the coefficient's scale sum |q| 0.7^k
    // (|w0| <= sqrt(2)/2); cfg4: dmax = 0.02, J = 20
    double dmax = 0.0;
    for (const double2& d : drift) dmax = std::max(dmax, std::hypot(d.x, d.y));
    int J = P;
    for (int j = 1; j <= P; ++j) {
        double c = 1.0;
        for (int t = 1; t <= j; ++t) c *= double(P - j + t) / t;  // C(P, j)
        if (c * std::pow(dmax / 0.7, j) < 1e-17) {
            J = j;
            break;
        }
    }
    pl.lat_shift_terms = J;
    std::vector<double> binom(51 * 51, 0.0);
    for (int k = 0; k <= 50; ++k) {
        binom[size_t(k) * 51] = 1.0;
        for (int i = 1; i <= k; ++i)
            binom[size_t(k) * 51 + i] = binom[size_t(k - 1) * 51 + i - 1] + (i <= k - 1 ? binom[size_t(k - 1) * 51 + i] : 0.0);
    }
    auto up = [](auto& d, const auto& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    };
    up(pl.lat_V, V);
    up(pl.lat_binom, binom);
    up(pl.lat_p2m_src, src);
    up(pl.lat_p2m_rows, rows);
    up(pl.lat_drift, drift);
    pl.lat_p2m_ncol = items;
    pl.lat_p2m = true;
}

// Decides whether the plan's leaves are translates of one pattern and, if
// so, builds the lattice schedule for the target leaves [lb, le): K, the
// neighbour table and the one-slot SymLeaf list of the finalize.  Called
// from build_sym_near on symmetric ("targets = nodes") Laplace plans whose
// targets are all matched.  VPG_LATTICE=0 disables the path.
bool build_lattice_near(Plan& pl, int64_t lb, int64_t le) {
    pl.lat = false;
    const char* ev = std::getenv("VPG_LATTICE");
    if (ev && std::atoi(ev) == 0) return false;
    if (pl.family != VPG_LAPLACE || pl.adaptive || pl.direct || !pl.matched || pl.nt != pl.ns) return false;
    const int L = pl.L;
    const int nb = 1 << L;
    const int64_t nleaf = int64_t(1) << (2 * L);
    const std::vector<int32_t>& so = pl.h_soff;
    // one point count, 64 / 128 / 256
    int m = 0;
    int64_t first = -1, nonempty = 0;
    for (int64_t b = 0; b < nleaf; ++b) {
        const int c = so[size_t(b) + 1] - so[size_t(b)];
        if (!c) continue;
        if (!m) {
            m = c;
            first = b;
        }
        if (c != m) return false;
        ++nonempty;
    }
    if (!(m == 64 || m == 128 || m == 256) || nonempty < 64) return false;
    // the coordinates, Morton-sorted (plan time only)
    std::vector<double2> xy(size_t(pl.ns));
    VPG_CUDA(cudaMemcpy(xy.data(), pl.src_sorted.p, sizeof(double2) * xy.size(), cudaMemcpyDeviceToHost));
    const double2* pat = xy.data() + so[size_t(first)];
    const int fx = int(squash2(uint32_t(first))), fy = int(squash2(uint32_t(first) >> 1));
    // lattice pitch from the farthest non-empty leaves in x and in y
    double px = 0.0, py = 0.0;
    int bestx = 0, besty = 0;
    for (int64_t b = 0; b < nleaf; ++b) {
        if (so[size_t(b) + 1] == so[size_t(b)]) continue;
        const int ix = int(squash2(uint32_t(b))) - fx, iy = int(squash2(uint32_t(b) >> 1)) - fy;
        const double2 p0 = xy[size_t(so[size_t(b)])];
        if (std::abs(ix) > std::abs(bestx)) {
            bestx = ix;
            px = (p0.x - pat[0].x) / ix;
        }
        if (std::abs(iy) > std::abs(besty)) {
            besty = iy;
            py = (p0.y - pat[0].y) / iy;
        }
    }
    if (bestx == 0 || besty == 0 || !(px > 0.0) || !(py > 0.0)) return false;
    // congruence on the actual coordinates: within a few ulp of pattern + translation
    double scale = std::max(std::fabs(pl.x0) + pl.side, std::fabs(pl.y0) + pl.side);
    const double tol = 16.0 * 2.220446049250313e-16 * scale;
    for (int64_t b = 0; b < nleaf; ++b) {
        if (so[size_t(b) + 1] == so[size_t(b)]) continue;
        const int ix = int(squash2(uint32_t(b))) - fx, iy = int(squash2(uint32_t(b) >> 1)) - fy;
        const double tx = ix * px, ty = iy * py;
        const double2* p = xy.data() + so[size_t(b)];
        for (int k = 0; k < m; ++k)
            if (std::fabs(p[k].x - (pat[k].x + tx)) > tol || std::fabs(p[k].y - (pat[k].y + ty)) > tol) return false;
    }
    // K_o on the device from the pattern's own coordinates
    {
        DBuf<double2> dpat;
        dpat.alloc(size_t(m));
        VPG_CUDA(cudaMemcpy(dpat.p, pat, sizeof(double2) * size_t(m), cudaMemcpyHostToDevice));
        pl.lat_K.alloc(size_t(9) * m * lat_la(m));
        lat_build_kernel<<<unsigned(pl.sm_count) * 4, 256>>>(dpat.p, m, px, py, pl.lat_K.p);
        VPG_LAUNCH_CHECK();
        VPG_CUDA(cudaDeviceSynchronize());
    }
    // target leaves of the range, their neighbours' charge runs, the finalize's leaves
    std::vector<int32_t> nbr;
    std::vector<SymLeaf> leaves;
    for (const LeafNear& ln : pl.h_leafnear) {
        const int64_t a = ln.leaf;
        if (a < lb || a >= le) continue;
        if (ln.t1 - ln.t0 != m) return false;  // every target matched (nt == ns, same leaves)
        const int ix = int(squash2(uint32_t(a))), iy = int(squash2(uint32_t(a) >> 1));
        const int64_t col = int64_t(leaves.size());
        for (int o = 0; o < 9; ++o) {
            const int jx = ix + o % 3 - 1, jy = iy + o / 3 - 1;
            int32_t src = -1;
            if (jx >= 0 && jy >= 0 && jx < nb && jy < nb) {
                const int64_t s = int64_t(mort(uint32_t(jx), uint32_t(jy)));
                if (so[size_t(s) + 1] > so[size_t(s)]) src = so[size_t(s)];
            }
            nbr.push_back(src);
        }
        leaves.push_back(SymLeaf{col * m, ln.t0, m, 1, ln.t1, ln.rfirst, ln.rcount, ln.lfirst, ln.lcount});
    }
    if (leaves.empty()) return false;
    pl.lat_ncol = int64_t(leaves.size());
    pl.lat_m = m;
    // the column tile with the fewest idle CTA-rounds (whole waves of sm_count tiles)
    int best_nt = 64;
    double best_cost = 1e300;
    for (int nt : {64, 56, 48, 40}) {
        const int64_t tiles = (pl.lat_ncol + nt - 1) / nt;
        const double cost = double((tiles + pl.sm_count - 1) / pl.sm_count) * (nt + 6.0);  // + per-tile overhead
        if (cost < best_cost) {
            best_cost = cost;
            best_nt = nt;
        }
    }
    pl.lat_nt = best_nt;
    auto up = [](auto& d, const auto& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    };
    up(pl.lat_nbr, nbr);
    up(pl.sym_leaves, leaves);
    pl.n_sym_leaves = pl.lat_ncol;
    pl.n_sym_tasks = 0;
    pl.sym_nparts = pl.lat_ncol * m;
    pl.sym_unmatched = false;
    pl.sym_hybrid = false;
    pl.n_hyb_chunks = 0;
    pl.sym_l2p_single = true;
    for (const SymLeaf& lf : leaves) pl.sym_l2p_single = pl.sym_l2p_single && lf.lcount == 1;
    pl.lat_pairs_exec = double(pl.lat_ncol) * 9.0 * double(m) * double(m);
    pl.lat_near_parts = pl.sym_nparts;
    build_lattice_p2m(pl, pat, first, px, py);
    if (pl.lat_p2m) pl.sym_nparts += pl.lat_p2m_ncol * kLatSRows;  // S scratch behind the near-field slots
    pl.sym = true;
    pl.lat = true;
    return true;
}

}  // namespace vpg
