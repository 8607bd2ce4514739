// Device-resident Davidson building blocks (reference: davidson.py).
//
// The reference driver keeps V, W as lists of N-vectors and makes many
// separate passes per iteration (V.w, Ritz vectors, residuals, a full Gram
// matrix, two sequential MGS sweeps).  Here every pass over the subspace is a
// single fused streaming kernel that reads each of the k basis vectors once
// per element and reduces its dot products deterministically (per-block
// partials, then an ordered sum) -- the subspace work is HBM-bound, so the
// number of passes over V/W is the cost that matters:
//
//   sbd_vdots            T[:, k-1] = V^T w                          (davidson.py:248-249)
//   sbd_residual_precond r = Y^T W - theta Y^T V, t = precond(r),   (davidson.py:252-258,
//                        |r|^2, |t|^2 and V^T t in the same pass      159-163, 278)
//   sbd_gs_update        t -= V c ; V^T t ; |t|^2  (one CGS pass;    (davidson.py:166-185)
//                        two calls = CGS2 reorthogonalisation)
//   sbd_rotate           thick restart V <- V Y_keep in place       (davidson.py:280-289)
//   sbd_jacobi           projected k x k eigensolve, one warp       (davidson.py:86-148)
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "sbd_internal.cuh"
#include "sbd_ptx.cuh"

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Reduce acc[0..K) over the block and store to partial[blockIdx.x * K + i].
template <int K>
__device__ __forceinline__ void block_partials(const double (&acc)[K], double *__restrict__ partial) {
    __shared__ double sm[kWarps][K];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        double v = warp_sum(acc[i]);
        if (lane == 0) sm[w][i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        double s = 0.0;
        for (int ww = 0; ww < kWarps; ++ww) s += sm[ww][i];
        partial[(i64)blockIdx.x * K + i] = s;
    }
}

// Ordered sum of per-block partials (deterministic).  Output slot i < k reads
// partial slot i; slot i >= k reads partial slot kfix + (i - k), so kernels
// can keep a compile-time accumulator layout for a runtime subspace size.
// One warp per output: lane l sums blocks l, l+32, ... in order, then a fixed
// shuffle tree -- the same order every call.
constexpr int kFinishBlocks = 24;  // x 4 warps >= the largest output count (2*64 + 9)
__global__ void finish_partials(const double *__restrict__ partial, int nblocks, int stride, int k, int kfix,
                                int cnt, double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += (gridDim.x * blockDim.x) >> 5) {
        const int src = i < k ? i : kfix + (i - k);
        double s = 0.0;
        for (int b = lane; b < nblocks; b += 32) s += partial[(i64)b * stride + src];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[i] = s;
    }
}

// Streaming over element "slots": with V2 a slot is a 16-byte pair of doubles
// (128-bit loads), otherwise one double.  Callers guarantee 16-byte aligned
// bases and even leading dimensions for V2; the odd tail element of a V2 run
// is folded in by thread 0 of block 0.
template <bool V2>
struct Slot {
    static constexpr int W = V2 ? 2 : 1;
    double v[2];
    __device__ __forceinline__ void load(const double *p, i64 s) {
        if (V2) {
            const double2 t = __ldg(reinterpret_cast<const double2 *>(p) + s);
            v[0] = t.x;
            v[1] = t.y;
        } else {
            v[0] = __ldg(p + s);
            v[1] = 0.0;
        }
    }
    __device__ __forceinline__ void load_cs(const double *p, i64 s) {
        if (V2) {
            const double2 t = __ldcs(reinterpret_cast<const double2 *>(p) + s);
            v[0] = t.x;
            v[1] = t.y;
        } else {
            v[0] = __ldcs(p + s);
            v[1] = 0.0;
        }
    }
    __device__ __forceinline__ void load_rw(const double *p, i64 s) {  // data written earlier in this kernel
        if (V2) {
            const double2 t = reinterpret_cast<const double2 *>(p)[s];
            v[0] = t.x;
            v[1] = t.y;
        } else {
            v[0] = p[s];
            v[1] = 0.0;
        }
    }
    __device__ __forceinline__ void store(double *p, i64 s) const {
        if (V2) reinterpret_cast<double2 *>(p)[s] = make_double2(v[0], v[1]);
        else p[s] = v[0];
    }
    __device__ __forceinline__ double dot(const Slot &o) const { return V2 ? fma(v[0], o.v[0], v[1] * o.v[1]) : v[0] * o.v[0]; }
};

// visit every slot once (grid-stride), then the scalar tail (n odd, V2) once
template <bool V2, class FS, class FT>
__device__ __forceinline__ void for_slots(i64 n, FS &&slot_fn, FT &&tail_fn) {
    const i64 ns = V2 ? n / 2 : n;
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += (i64)gridDim.x * blockDim.x) slot_fn(s);
    if (V2 && (n & 1) && blockIdx.x == 0 && threadIdx.x == 0) tail_fn(n - 1);
}

template <int K, bool V2>
__global__ void __launch_bounds__(kBlock) vdots_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                       const double *__restrict__ w, double *__restrict__ partial) {
    double acc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] = 0.0;
    const i64 ldvs = V2 ? ldv / 2 : ldv;
    for_slots<V2>(n, [&](i64 s) {
        Slot<V2> ws;
        ws.load_cs(w, s);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                Slot<V2> vs;
                vs.load_cs(V + i * ldv, s);
                acc[i] += vs.dot(ws);
            }
    }, [&](i64 e) {
        const double we = w[e];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) acc[i] = fma(V[i * ldv + e], we, acc[i]);
    });
    (void)ldvs;
    block_partials<K>(acc, partial);
}

// out[i] = V_i . w, out[K + i] = V_i . u  (one pass over V, two right-hand sides)
template <int K, bool V2>
__global__ void __launch_bounds__(kBlock) vdots2_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                        const double *__restrict__ w, const double *__restrict__ u,
                                                        double *__restrict__ partial) {
    double acc[2 * K];
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) acc[i] = 0.0;
    for_slots<V2>(n, [&](i64 s) {
        Slot<V2> ws, us;
        ws.load_cs(w, s);
        us.load(u, s);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                Slot<V2> vs;
                vs.load_cs(V + i * ldv, s);
                acc[i] += vs.dot(ws);
                acc[K + i] += vs.dot(us);
            }
    }, [&](i64 e) {
        const double we = w[e], ue = u[e];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                const double v = V[i * ldv + e];
                acc[i] = fma(v, we, acc[i]);
                acc[K + i] = fma(v, ue, acc[K + i]);
            }
    });
    block_partials<2 * K>(acc, partial);
}

// Ritz residual, preconditioner and projections (M = compile-time bound on roots)
template <int K, int M, bool V2>
__global__ void __launch_bounds__(kBlock)
residual_kernel(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
                const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
                const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
                double *__restrict__ partial) {
    __shared__ double ys[64 * 8];
    __shared__ double th[8];
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    if (threadIdx.x < m) th[threadIdx.x] = theta[threadIdx.x];
    __syncthreads();
    // accumulator layout: [0,K) V^T t_jp | K: |t_jp|^2 | K+1+j: |r_j|^2
    double acc[K + 1 + M];
#pragma unroll
    for (int i = 0; i < K + 1 + M; ++i) acc[i] = 0.0;
    auto element = [&](const double (&u)[M], const double (&wy)[M], double d, double *tout, i64 ldt_, i64 pos,
                       double &tj_out) {
        double tj = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if (j < m) {
                const double r = wy[j] - th[j] * u[j];
                acc[K + 1 + j] = fma(r, r, acc[K + 1 + j]);
                const double g = d - th[j];
                const double den = (g >= 0.0 ? 1.0 : -1.0) * fmax(fabs(g), delta);  // davidson.py:159-163
                const double t = r / den;
                tout[j * ldt_ + pos] = t;
                if (j == jp) tj = t;
            }
        }
        acc[K] = fma(tj, tj, acc[K]);
        tj_out = tj;
    };
    for_slots<V2>(n, [&](i64 s) {
        double u[2][M], wy[2][M];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < M; ++j) u[h][j] = wy[h][j] = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (i < k) {
                Slot<V2> vs, wsl;
                vs.load(V + i * ldv, s);
                wsl.load_cs(W + i * ldv, s);
#pragma unroll
                for (int j = 0; j < M; ++j)
                    if (j < m) {
                        const double yij = ys[i * m + j];
#pragma unroll
                        for (int h = 0; h < Slot<V2>::W; ++h) {
                            u[h][j] = fma(yij, vs.v[h], u[h][j]);
                            wy[h][j] = fma(yij, wsl.v[h], wy[h][j]);
                        }
                    }
            }
        }
        Slot<V2> ds;
        ds.load(diag, s);
        double tjv[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < Slot<V2>::W; ++h) element(u[h], wy[h], ds.v[h], T, ldt, (V2 ? 2 * s : s) + h, tjv[h]);
        Slot<V2> ts;
        ts.v[0] = tjv[0];
        ts.v[1] = tjv[1];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                Slot<V2> vs;
                vs.load(V + i * ldv, s);  // second touch: L1
                acc[i] += vs.dot(ts);
            }
    }, [&](i64 e) {
        double u[M], wy[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = wy[j] = 0.0;
        for (int i = 0; i < k; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j)
                if (j < m) {
                    u[j] = fma(ys[i * m + j], V[i * ldv + e], u[j]);
                    wy[j] = fma(ys[i * m + j], W[i * ldv + e], wy[j]);
                }
        double tj;
        element(u, wy, diag[e], T, ldt, e, tj);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) acc[i] = fma(V[i * ldv + e], tj, acc[i]);
    });
    block_partials<K + 1 + M>(acc, partial);
}

// t -= sum_i c_i V_i ; then partial dots V_i . t (i < kdot) and |t|^2 (slot K)
template <int K, bool V2>
__global__ void __launch_bounds__(kBlock) gs_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                    const double *__restrict__ c, int kdot, double *__restrict__ t,
                                                    double *__restrict__ partial) {
    __shared__ double cs[K > 0 ? K : 1];
    for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
    __syncthreads();
    double acc[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) acc[i] = 0.0;
    for_slots<V2>(n, [&](i64 s) {
        Slot<V2> ts;
        ts.load_rw(t, s);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                Slot<V2> vs;
                vs.load(V + i * ldv, s);
#pragma unroll
                for (int h = 0; h < Slot<V2>::W; ++h) ts.v[h] = fma(-cs[i], vs.v[h], ts.v[h]);
            }
        ts.store(t, s);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < kdot) {
                Slot<V2> vs;
                vs.load(V + i * ldv, s);  // second touch: L1
                acc[i] += vs.dot(ts);
            }
        acc[K] += ts.dot(ts);
    }, [&](i64 e) {
        double te = t[e];
        for (int i = 0; i < k; ++i) te = fma(-cs[i], V[i * ldv + e], te);
        t[e] = te;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < kdot) acc[i] = fma(V[i * ldv + e], te, acc[i]);
        acc[K] = fma(te, te, acc[K]);
    });
    block_partials<K + 1>(acc, partial);
}

// ---------------------------------------------------------------------------
// Tile kernels (the aligned fast path).  A CTA walks tiles of TT contiguous
// elements; its 8 warps split the k basis vectors (warp w owns vectors w,
// w+8, ...), and each lane issues QD independent 128-bit loads per vector, so
// a warp has QD*512 B in flight per vector with O(k/8) accumulators -- the
// register pressure of a per-element design is gone.  Cross-warp sums over
// the vectors (t - V c, Y^T V, Y^T W) go through shared memory.  Requires
// 16-byte aligned bases and even leading dimensions (the Python driver
// allocates that way); the per-element kernels above stay as the fallback.
constexpr int kWarpsT = kBlock / 32;

__device__ __forceinline__ double2 ld2(const double *__restrict__ p, i64 e, i64 n) {
    // p + e is 16-byte aligned (e even); elements >= n read as 0
    if (e + 1 < n) return __ldcs(reinterpret_cast<const double2 *>(p + e));
    if (e < n) return make_double2(__ldcs(p + e), 0.0);
    return make_double2(0.0, 0.0);
}
__device__ __forceinline__ double2 ld2_keep(const double *__restrict__ p, i64 e, i64 n) {
    if (e + 1 < n) return __ldg(reinterpret_cast<const double2 *>(p + e));
    if (e < n) return make_double2(__ldg(p + e), 0.0);
    return make_double2(0.0, 0.0);
}
__device__ __forceinline__ double dot2(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

// out[i] = V_i . w, out[K + i] = V_i . u
template <int K>
__global__ void __launch_bounds__(kBlock) vdots2_tile(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                      const double *__restrict__ w, const double *__restrict__ u,
                                                      double *__restrict__ partial) {
    constexpr int TT = 1024, QD = TT / 64, KW = (K + kWarpsT - 1) / kWarpsT;
    __shared__ double2 ws[TT / 2], us[TT / 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double aw[KW], au[KW];
#pragma unroll
    for (int a = 0; a < KW; ++a) aw[a] = au[a] = 0.0;
    for (i64 base = (i64)blockIdx.x * TT; base < n; base += (i64)gridDim.x * TT) {
        const i64 rem = n - base;
        for (int d = threadIdx.x; d < TT / 2; d += blockDim.x) {
            ws[d] = ld2(w + base, 2 * d, rem);
            us[d] = ld2_keep(u + base, 2 * d, rem);
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < KW; ++a) {
            const int i = warp + kWarpsT * a;
            if (i < k) {
                const double *vi = V + i * ldv + base;
                double2 v[QD];
#pragma unroll
                for (int q = 0; q < QD; ++q) v[q] = ld2(vi, 2 * (lane + 32 * q), rem);
#pragma unroll
                for (int q = 0; q < QD; ++q) {
                    aw[a] += dot2(v[q], ws[lane + 32 * q]);
                    au[a] += dot2(v[q], us[lane + 32 * q]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < KW; ++a) {
        const int i = warp + kWarpsT * a;
        const double sw = warp_sum(aw[a]), su = warp_sum(au[a]);
        if (lane == 0 && i < K) {
            partial[(i64)blockIdx.x * 2 * K + i] = i < k ? sw : 0.0;
            partial[(i64)blockIdx.x * 2 * K + K + i] = i < k ? su : 0.0;
        }
    }
}

// t -= V c ; dots V_i . t (i < kdot) ; |t|^2  -> partial[b * (K+1) + ...]
template <int K>
__global__ void __launch_bounds__(kBlock) gs_tile(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                  const double *__restrict__ c, int kdot, double *__restrict__ t,
                                                  double *__restrict__ partial) {
    constexpr int TT = 512, QD = TT / 64, KW = (K + kWarpsT - 1) / kWarpsT;
    __shared__ double2 part[kWarpsT][TT / 2];
    __shared__ double2 ts[TT / 2];
    __shared__ double cs[K];
    __shared__ double nrm[kWarpsT];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
    double acc[KW];
#pragma unroll
    for (int a = 0; a < KW; ++a) acc[a] = 0.0;
    double n2 = 0.0;
    __syncthreads();
    for (i64 base = (i64)blockIdx.x * TT; base < n; base += (i64)gridDim.x * TT) {
        const i64 rem = n - base;
        // phase 1: warp partial of sum_i c_i V_i over its vectors
        double2 s[QD];
#pragma unroll
        for (int q = 0; q < QD; ++q) s[q] = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < KW; ++a) {
            const int i = warp + kWarpsT * a;
            if (i < k) {
                const double *vi = V + i * ldv + base;
                const double ci = cs[i];
#pragma unroll
                for (int q = 0; q < QD; ++q) {
                    const double2 v = ld2_keep(vi, 2 * (lane + 32 * q), rem);
                    s[q].x = fma(ci, v.x, s[q].x);
                    s[q].y = fma(ci, v.y, s[q].y);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < QD; ++q) part[warp][lane + 32 * q] = s[q];
        __syncthreads();
        // combine: t_new = t - sum over warps
        for (int d = threadIdx.x; d < TT / 2; d += blockDim.x) {
            const i64 e = base + 2 * d;
            double2 tv = make_double2(0.0, 0.0);
            if (e + 1 < n) tv = *reinterpret_cast<const double2 *>(t + e);
            else if (e < n) tv.x = t[e];
#pragma unroll
            for (int ww = 0; ww < kWarpsT; ++ww) {
                tv.x -= part[ww][d].x;
                tv.y -= part[ww][d].y;
            }
            if (e + 1 < n) *reinterpret_cast<double2 *>(t + e) = tv;
            else if (e < n) t[e] = tv.x;
            if (e >= n) tv.x = 0.0;
            if (e + 1 >= n) tv.y = 0.0;
            ts[d] = tv;
            n2 += dot2(tv, tv);
        }
        __syncthreads();
        // phase 2: dots with the updated t (V tile re-read: L1/L2)
        if (kdot > 0) {
#pragma unroll
            for (int a = 0; a < KW; ++a) {
                const int i = warp + kWarpsT * a;
                if (i < kdot) {
                    const double *vi = V + i * ldv + base;
#pragma unroll
                    for (int q = 0; q < QD; ++q) acc[a] += dot2(ld2_keep(vi, 2 * (lane + 32 * q), rem), ts[lane + 32 * q]);
                }
            }
        }
        __syncthreads();
    }
    n2 = warp_sum(n2);
    if (lane == 0) nrm[warp] = n2;
#pragma unroll
    for (int a = 0; a < KW; ++a) {
        const int i = warp + kWarpsT * a;
        const double sa = warp_sum(acc[a]);
        if (lane == 0 && i < K) partial[(i64)blockIdx.x * (K + 1) + i] = i < kdot ? sa : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int ww = 0; ww < kWarpsT; ++ww) s += nrm[ww];
        partial[(i64)blockIdx.x * (K + 1) + K] = s;
    }
}

// Ritz residuals, preconditioned corrections T_j and projections V^T t_jp.
// partial layout per block (stride K + 1 + M): [0,K) dots | K: |t_jp|^2 | K+1+j: |r_j|^2
template <int K, int M>
__global__ void __launch_bounds__(kBlock)
residual_tile(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
              const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
              const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
              double *__restrict__ partial) {
    constexpr int TT = 512 / M, QD = TT / 64 > 0 ? TT / 64 : 1, KW = (K + kWarpsT - 1) / kWarpsT;
    extern __shared__ double2 rsm[];
    double2 *pu = rsm;                                  // [kWarpsT][M][TT/2]
    double2 *pw = rsm + kWarpsT * M * (TT / 2);         // [kWarpsT][M][TT/2]
    double2 *ts = pw + kWarpsT * M * (TT / 2);          // [TT/2]
    __shared__ double ys[64 * 8];
    __shared__ double th[8];
    __shared__ double red[kWarpsT][M + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    if (threadIdx.x < m) th[threadIdx.x] = theta[threadIdx.x];
    double acc[KW];
#pragma unroll
    for (int a = 0; a < KW; ++a) acc[a] = 0.0;
    double rn2[M], tn2 = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = 0.0;
    __syncthreads();
    for (i64 base = (i64)blockIdx.x * TT; base < n; base += (i64)gridDim.x * TT) {
        const i64 rem = n - base;
        double2 u[M][QD], wy[M][QD];
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
            for (int q = 0; q < QD; ++q) u[j][q] = wy[j][q] = make_double2(0.0, 0.0);
        const bool lane_on = 2 * lane < TT;  // M = 8: a tile is 64 elements = 32 pairs
#pragma unroll
        for (int a = 0; a < KW; ++a) {
            const int i = warp + kWarpsT * a;
            if (i < k && lane_on) {
                const double *vi = V + i * ldv + base, *wi = W + i * ldv + base;
                double2 v[QD], x[QD];
#pragma unroll
                for (int q = 0; q < QD; ++q) {
                    v[q] = ld2_keep(vi, 2 * (lane + 32 * q), rem);
                    x[q] = ld2(wi, 2 * (lane + 32 * q), rem);
                }
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    if (j < m) {
                        const double y = ys[i * m + j];
#pragma unroll
                        for (int q = 0; q < QD; ++q) {
                            u[j][q].x = fma(y, v[q].x, u[j][q].x);
                            u[j][q].y = fma(y, v[q].y, u[j][q].y);
                            wy[j][q].x = fma(y, x[q].x, wy[j][q].x);
                            wy[j][q].y = fma(y, x[q].y, wy[j][q].y);
                        }
                    }
                }
            }
        }
        if (lane_on) {
#pragma unroll
            for (int j = 0; j < M; ++j)
#pragma unroll
                for (int q = 0; q < QD; ++q) {
                    pu[(warp * M + j) * (TT / 2) + lane + 32 * q] = u[j][q];
                    pw[(warp * M + j) * (TT / 2) + lane + 32 * q] = wy[j][q];
                }
        }
        __syncthreads();
        for (int d = threadIdx.x; d < TT / 2; d += blockDim.x) {
            const i64 e = base + 2 * d;
            const double2 dg = ld2_keep(diag, e, n);
            double2 tj = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                if (j < m) {
                    double2 uu = make_double2(0.0, 0.0), ww2 = make_double2(0.0, 0.0);
#pragma unroll
                    for (int w2 = 0; w2 < kWarpsT; ++w2) {
                        const double2 a1 = pu[(w2 * M + j) * (TT / 2) + d], b1 = pw[(w2 * M + j) * (TT / 2) + d];
                        uu.x += a1.x;
                        uu.y += a1.y;
                        ww2.x += b1.x;
                        ww2.y += b1.y;
                    }
                    // r = Y^T W - theta Y^T V ; t = r / (sign(d - theta) max(|d - theta|, delta))
                    const double rx = ww2.x - th[j] * uu.x, ry = ww2.y - th[j] * uu.y;
                    const double gx = dg.x - th[j], gy = dg.y - th[j];
                    const double tx = rx / ((gx >= 0.0 ? 1.0 : -1.0) * fmax(fabs(gx), delta));
                    const double ty = ry / ((gy >= 0.0 ? 1.0 : -1.0) * fmax(fabs(gy), delta));
                    double *tr = T + j * ldt;
                    if (e + 1 < n) {
                        *reinterpret_cast<double2 *>(tr + e) = make_double2(tx, ty);
                        rn2[j] += rx * rx + ry * ry;
                    } else if (e < n) {
                        tr[e] = tx;
                        rn2[j] += rx * rx;
                    }
                    if (j == jp) tj = make_double2(e < n ? tx : 0.0, e + 1 < n ? ty : 0.0);
                }
            }
            ts[d] = tj;
            tn2 += dot2(tj, tj);
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < KW; ++a) {
            const int i = warp + kWarpsT * a;
            if (i < k && lane_on) {
                const double *vi = V + i * ldv + base;
#pragma unroll
                for (int q = 0; q < QD; ++q) acc[a] += dot2(ld2_keep(vi, 2 * (lane + 32 * q), rem), ts[lane + 32 * q]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < KW; ++a) {
        const int i = warp + kWarpsT * a;
        const double s = warp_sum(acc[a]);
        if (lane == 0 && i < K) partial[(i64)blockIdx.x * (K + 1 + M) + i] = i < k ? s : 0.0;
    }
    tn2 = warp_sum(tn2);
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = warp_sum(rn2[j]);
    if (lane == 0) {
        red[warp][0] = tn2;
#pragma unroll
        for (int j = 0; j < M; ++j) red[warp][1 + j] = rn2[j];
    }
    __syncthreads();
    if (threadIdx.x <= M) {
        double s = 0.0;
        for (int ww = 0; ww < kWarpsT; ++ww) s += red[ww][threadIdx.x];
        partial[(i64)blockIdx.x * (K + 1 + M) + K + threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// TMA-pipelined kernels (aligned fast path for the multi-phase passes).
// A CTA owns a strided set of tiles of TT elements.  For each tile one thread
// issues 1-D bulk copies (cp.async.bulk) of every vector slice the tile
// needs into a shared-memory stage, counted on that stage's mbarrier; two
// stages alternate, so tile i+1 streams in from HBM while tile i is computed
// entirely out of shared memory (no second global touch, no register
// staging).  Stage size is ~64 KB, i.e. TT = 8192 / (#vectors per tile).

// even tile length so that nvec slices of one stage take ~64 KB (<= 1024 elements)
__host__ __device__ constexpr int tma_tile(int nvec) {
    return ((8192 / nvec) < 1024 ? (8192 / nvec) : 1024) & ~1;
}
// elements per lane needed by residual_tma<K> over the k range dispatch_k maps to K
__host__ __device__ constexpr int resid_epl(int K) {
    return (tma_tile(2 * (K <= 8 ? 1 : K / 2 + 1) + 1) + 31) / 32;
}

struct TmaPipe {
    uint64_t *bar;  // [2]
    __device__ void init() {
        if (threadIdx.x == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            mbar_fence_init();
        }
        __syncthreads();
    }
};

// copy `cnt` doubles starting at src (16-B aligned) to dst; the odd last
// element (if any) is loaded by plain loads later -- returns bytes issued
__device__ __forceinline__ uint32_t bulk_bytes(i64 cnt) { return (uint32_t)((cnt & ~(i64)1) * 8); }

// t_new = t - V c ; out = scale * t_new (out may alias t) ; dots V_i.t_new (i<kdot) ; |t_new|^2
template <int K>
__global__ void __launch_bounds__(kBlock)
gs_tma(const double *__restrict__ V, int k, i64 ldv, i64 n, const double *__restrict__ c, int kdot,
       const double *t, double *out, const double *__restrict__ scale, double *__restrict__ partial) {
    constexpr int KW = (K + kWarpsT - 1) / kWarpsT;
    const int TTA = tma_tile(k + 1);  // ~64 KB of slices per stage, even length
    extern __shared__ __align__(128) unsigned char gsm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(gsm);
    double *stage0 = reinterpret_cast<double *>(gsm + 128);
    const i64 sstride = (i64)(k + 1) * TTA;  // doubles per stage: k V slices + t slice
    __shared__ double cs[K];
    __shared__ double nrm[kWarpsT];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
    const double sc = scale ? *scale : 1.0;
    TmaPipe pipe{bar};
    pipe.init();
    const i64 ntiles = (n + TTA - 1) / TTA;
    auto issue = [&](i64 tile, int s) {
        const i64 base = tile * TTA, cnt = min((i64)TTA, n - base);
        const uint32_t b = bulk_bytes(cnt);
        double *st = stage0 + s * sstride;
        if (b) {
            mbar_arrive_expect_tx(&bar[s], b * (uint32_t)(k + 1));
            for (int i = 0; i < k; ++i) tma_load_1d(st + (i64)i * TTA, V + i * ldv + base, b, &bar[s]);
            tma_load_1d(st + (i64)k * TTA, t + base, b, &bar[s]);
        } else {
            mbar_arrive_expect_tx(&bar[s], 0);
        }
    };
    double acc[KW];
#pragma unroll
    for (int a = 0; a < KW; ++a) acc[a] = 0.0;
    double n2 = 0.0;
    i64 tile = blockIdx.x;
    if (threadIdx.x == 0) {
        if (tile < ntiles) issue(tile, 0);
        if (tile + gridDim.x < ntiles) issue(tile + gridDim.x, 1);
    }
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        const i64 base = tile * TTA, cnt = min((i64)TTA, n - base);
        double *st = stage0 + s * sstride;
        mbar_wait(&bar[s], (uint32_t)((it >> 1) & 1));
        if (cnt & 1) {  // odd tail element: plain loads
            const i64 e = cnt - 1;
            if (threadIdx.x == 0) {
                for (int i = 0; i < k; ++i) st[(i64)i * TTA + e] = V[i * ldv + base + e];
                st[(i64)k * TTA + e] = t[base + e];
            }
            __syncthreads();
        }
        double *ts = st + (i64)k * TTA;
        for (i64 e = threadIdx.x; e < cnt; e += blockDim.x) {
            double v = ts[e];
            for (int i = 0; i < k; ++i) v = fma(-cs[i], st[(i64)i * TTA + e], v);
            ts[e] = v;
            out[base + e] = v * sc;
            n2 = fma(v, v, n2);
        }
        __syncthreads();
        if (kdot > 0) {
#pragma unroll
            for (int a = 0; a < KW; ++a) {
                const int i = warp + kWarpsT * a;
                if (i < kdot) {
                    const double *vi = st + (i64)i * TTA;
                    double sacc = 0.0;
                    for (i64 e = lane; e < cnt; e += 32) sacc = fma(vi[e], ts[e], sacc);
                    acc[a] += sacc;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, s);
    }
    n2 = warp_sum(n2);
    if (lane == 0) nrm[warp] = n2;
#pragma unroll
    for (int a = 0; a < KW; ++a) {
        const int i = warp + kWarpsT * a;
        const double sa = warp_sum(acc[a]);
        if (lane == 0 && i < K) partial[(i64)blockIdx.x * (K + 1) + i] = i < kdot ? sa : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int ww = 0; ww < kWarpsT; ++ww) sum += nrm[ww];
        partial[(i64)blockIdx.x * (K + 1) + K] = sum;
    }
}

// Ritz residual + preconditioner + projections, TMA-fed (stage: k V + k W + diag
// slices).  Phase 1 is split over all 8 warps (warp w sums its vectors
// i = w, w+8, ... for every element; lanes stride the tile), partial sums are
// combined through shared memory, then the element-wise residual /
// preconditioner, then the warp-split projections V_i . t_jp.
template <int K, int M>
__global__ void __launch_bounds__(kBlock)
residual_tma(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
             const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
             const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
             double *__restrict__ partial) {
    constexpr int KW = (K + kWarpsT - 1) / kWarpsT;
    constexpr int EPL = resid_epl(K);  // elements per lane in the warp-split phases (max over k)
    const int TTA = tma_tile(2 * k + 1);
    extern __shared__ __align__(128) unsigned char rsm2[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(rsm2);
    double *stage0 = reinterpret_cast<double *>(rsm2 + 128);
    const i64 sstride = (i64)(2 * k + 1) * TTA;
    double *ts = stage0 + 2 * sstride;                 // [TTA] correction of the target root
    double *pu = ts + TTA;                             // [kWarpsT][M][TTA]
    double *pw = pu + (size_t)kWarpsT * M * TTA;       // [kWarpsT][M][TTA]
    __shared__ double ys[64 * 8];
    __shared__ double th[8];
    __shared__ double red[kWarpsT][M + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    if (threadIdx.x < m) th[threadIdx.x] = theta[threadIdx.x];
    TmaPipe pipe{bar};
    pipe.init();
    const i64 ntiles = (n + TTA - 1) / TTA;
    auto issue = [&](i64 tile, int s) {
        const i64 base = tile * TTA, cnt = min((i64)TTA, n - base);
        const uint32_t b = bulk_bytes(cnt);
        double *st = stage0 + s * sstride;
        if (b) {
            mbar_arrive_expect_tx(&bar[s], b * (uint32_t)(2 * k + 1));
            for (int i = 0; i < k; ++i) {
                tma_load_1d(st + (i64)i * TTA, V + i * ldv + base, b, &bar[s]);
                tma_load_1d(st + (i64)(k + i) * TTA, W + i * ldv + base, b, &bar[s]);
            }
            tma_load_1d(st + (i64)(2 * k) * TTA, diag + base, b, &bar[s]);
        } else {
            mbar_arrive_expect_tx(&bar[s], 0);
        }
    };
    double acc[KW];
#pragma unroll
    for (int a = 0; a < KW; ++a) acc[a] = 0.0;
    double rn2[M], tn2 = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = 0.0;
    i64 tile = blockIdx.x;
    if (threadIdx.x == 0) {
        if (tile < ntiles) issue(tile, 0);
        if (tile + gridDim.x < ntiles) issue(tile + gridDim.x, 1);
    }
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        const i64 base = tile * TTA, cnt = min((i64)TTA, n - base);
        double *st = stage0 + s * sstride;
        mbar_wait(&bar[s], (uint32_t)((it >> 1) & 1));
        if (cnt & 1) {
            const i64 e = cnt - 1;
            if (threadIdx.x == 0) {
                for (int i = 0; i < k; ++i) {
                    st[(i64)i * TTA + e] = V[i * ldv + base + e];
                    st[(i64)(k + i) * TTA + e] = W[i * ldv + base + e];
                }
                st[(i64)(2 * k) * TTA + e] = diag[base + e];
            }
            __syncthreads();
        }
        // phase 1: per-warp partial Y^T V and Y^T W over the warp's vectors
        {
            double u[EPL][M], wy[EPL][M];
#pragma unroll
            for (int q = 0; q < EPL; ++q)
#pragma unroll
                for (int j = 0; j < M; ++j) u[q][j] = wy[q][j] = 0.0;
#pragma unroll
            for (int a = 0; a < KW; ++a) {
                const int i = warp + kWarpsT * a;
                if (i < k) {
                    const double *vi = st + (i64)i * TTA, *wi = st + (i64)(k + i) * TTA;
                    double yv[M];
#pragma unroll
                    for (int j = 0; j < M; ++j) yv[j] = j < m ? ys[i * m + j] : 0.0;
#pragma unroll
                    for (int q = 0; q < EPL; ++q) {
                        const int e = lane + 32 * q;
                        if (e < TTA) {
                            const double v = vi[e], w = wi[e];
#pragma unroll
                            for (int j = 0; j < M; ++j) {
                                u[q][j] = fma(yv[j], v, u[q][j]);
                                wy[q][j] = fma(yv[j], w, wy[q][j]);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < EPL; ++q) {
                const int e = lane + 32 * q;
                if (e < TTA) {
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        pu[((size_t)warp * M + j) * TTA + e] = u[q][j];
                        pw[((size_t)warp * M + j) * TTA + e] = wy[q][j];
                    }
                }
            }
        }
        __syncthreads();
        // phase 1b: combine, residual, preconditioner (davidson.py:159-163,257)
        for (i64 e = threadIdx.x; e < cnt; e += blockDim.x) {
            const double d = st[(i64)(2 * k) * TTA + e];
            double tj = 0.0;
#pragma unroll
            for (int j = 0; j < M; ++j) {
                if (j < m) {
                    double uu = 0.0, ww = 0.0;
#pragma unroll
                    for (int w2 = 0; w2 < kWarpsT; ++w2) {
                        uu += pu[((size_t)w2 * M + j) * TTA + e];
                        ww += pw[((size_t)w2 * M + j) * TTA + e];
                    }
                    const double r = ww - th[j] * uu;
                    rn2[j] = fma(r, r, rn2[j]);
                    const double g = d - th[j];
                    const double t = r / ((g >= 0.0 ? 1.0 : -1.0) * fmax(fabs(g), delta));
                    T[j * ldt + base + e] = t;
                    if (j == jp) tj = t;
                }
            }
            ts[e] = tj;
            tn2 = fma(tj, tj, tn2);
        }
        __syncthreads();
        // phase 2: projections V_i . t_jp (warp-split)
#pragma unroll
        for (int a = 0; a < KW; ++a) {
            const int i = warp + kWarpsT * a;
            if (i < k) {
                const double *vi = st + (i64)i * TTA;
                double sacc = 0.0;
#pragma unroll
                for (int q = 0; q < EPL; ++q) {
                    const int e = lane + 32 * q;
                    if (e < cnt) sacc = fma(vi[e], ts[e], sacc);
                }
                acc[a] += sacc;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, s);
    }
#pragma unroll
    for (int a = 0; a < KW; ++a) {
        const int i = warp + kWarpsT * a;
        const double sa = warp_sum(acc[a]);
        if (lane == 0 && i < K) partial[(i64)blockIdx.x * (K + 1 + M) + i] = i < k ? sa : 0.0;
    }
    tn2 = warp_sum(tn2);
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = warp_sum(rn2[j]);
    if (lane == 0) {
        red[warp][0] = tn2;
#pragma unroll
        for (int j = 0; j < M; ++j) red[warp][1 + j] = rn2[j];
    }
    __syncthreads();
    if (threadIdx.x <= M) {
        double sum = 0.0;
        for (int ww = 0; ww < kWarpsT; ++ww) sum += red[ww][threadIdx.x];
        partial[(i64)blockIdx.x * (K + 1 + M) + K + threadIdx.x] = sum;
    }
}

__global__ void scale_copy_kernel(const double *__restrict__ src, double *__restrict__ dst, i64 n,
                                  const double *__restrict__ s) {
    const double f = *s;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x)
        dst[e] = src[e] * f;
}

// in place: V[:, j] <- sum_i Y[i, j] V[:, i]  for j < keep (per element independent)
template <int K>
__global__ void __launch_bounds__(kBlock) rotate_kernel(double *__restrict__ V, int k, i64 ldv, i64 n,
                                                        const double *__restrict__ Y, int keep) {
    __shared__ double ys[K * K];
    for (int i = threadIdx.x; i < k * keep; i += blockDim.x) ys[i] = Y[i];
    __syncthreads();
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double v[K];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) v[i] = V[i * ldv + e];
        for (int j = 0; j < keep; ++j) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i < k) s = fma(ys[i * keep + j], v[i], s);
            V[j * ldv + e] = s;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) combine_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                         const double *__restrict__ Y, int m, double *__restrict__ U,
                                                         i64 ldu) {
    __shared__ double ys[K * 8];
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    __syncthreads();
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                const double v = V[i * ldv + e];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < m) u[j] = fma(ys[i * m + j], v, u[j]);
            }
        for (int j = 0; j < m; ++j) U[j * ldu + e] = u[j];
    }
}

// Jacobi eigensolver of the projected matrix (davidson.py:86-148): same
// rotation formulas, symmetrisation, stopping rule (off-norm <= 1e-14 ||A||_F
// at a sweep start) and stable ascending output order as the reference, but
// with the parallel (round-robin tournament) ordering: each step rotates
// kk/2 disjoint pairs at once (rows, then columns, of one CTA), so a sweep is
// kk-1 steps instead of k(k-1)/2 sequential rotations.  Eigenvalues agree
// with the cyclic order to rounding; eigenvector signs are arbitrary in both.
constexpr int kJacMax = 64;
constexpr int kJacThreads = 256;
__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(const double *__restrict__ Ain, int k, int lda,
                                                             double *__restrict__ evals, double *__restrict__ evecs,
                                                             int max_sweeps, int *__restrict__ info) {
    extern __shared__ double jsm[];
    double(*a)[kJacMax + 1] = reinterpret_cast<double(*)[kJacMax + 1]>(jsm);
    double(*v)[kJacMax + 1] = reinterpret_cast<double(*)[kJacMax + 1]>(jsm + kJacMax * (kJacMax + 1));
    double *rc = jsm + 2 * kJacMax * (kJacMax + 1);  // per pair: c, s, new a_pp, new a_qq  [4][kJacMax/2]
    int *order = reinterpret_cast<int *>(rc + 4 * (kJacMax / 2));
    int *pp = order + kJacMax;                       // pair members [2][kJacMax/2]
    __shared__ double red[kJacThreads / 32];
    __shared__ int stop;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kk = (k + 1) & ~1, np = kk / 2;  // even size (index k is a phantom when k is odd)
    for (int idx = tid; idx < k * k; idx += kJacThreads) {
        const int p = idx / k, q = idx % k;
        a[p][q] = (Ain[p * lda + q] + Ain[q * lda + p]) / 2.0;
        v[p][q] = p == q ? 1.0 : 0.0;
    }
    __syncthreads();
    double fro = 0.0;
    for (int idx = tid; idx < k * k; idx += kJacThreads) fro = fma(a[idx / k][idx % k], a[idx / k][idx % k], fro);
    fro = warp_sum(fro);
    if (lane == 0) red[warp] = fro;
    __syncthreads();
    if (tid == 0) {
        double f = 0.0;
        for (int w = 0; w < kJacThreads / 32; ++w) f += red[w];
        red[0] = f;
    }
    __syncthreads();
    const double tol = 1e-14 * sqrt(red[0]);
    __syncthreads();
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        double off = 0.0;
        for (int idx = tid; idx < k * k; idx += kJacThreads) {
            const int p = idx / k, q = idx % k;
            if (q > p) off += 2.0 * a[p][q] * a[p][q];
        }
        off = warp_sum(off);
        if (lane == 0) red[warp] = off;
        __syncthreads();
        if (tid == 0) {
            double f = 0.0;
            for (int w = 0; w < kJacThreads / 32; ++w) f += red[w];
            stop = sqrt(f) <= tol;
        }
        __syncthreads();
        if (stop) break;
        for (int step = 0; step < kk - 1; ++step) {
            // round robin: position 0 fixed, positions 1..kk-1 rotate by `step`
            if (tid < np) {
                auto at = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + step) % (kk - 1); };
                int p = at(tid), q = at(kk - 1 - tid);
                if (p > q) { const int t = p; p = q; q = t; }
                pp[tid] = p;
                pp[np + tid] = q;
                double c = 1.0, sn = 0.0, npp = 0.0, nqq = 0.0;
                int act = 0;
                if (q < k) {
                    const double apq = a[p][q];
                    if (apq != 0.0) {
                        act = 1;
                        const double app = a[p][p], aqq = a[q][q];
                        const double theta = (aqq - app) / (2.0 * apq);
                        double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                        if (theta < 0.0) t = -t;
                        c = 1.0 / sqrt(t * t + 1.0);
                        sn = t * c;
                        npp = app - t * apq;
                        nqq = aqq + t * apq;
                    }
                }
                rc[tid] = c;
                rc[kJacMax / 2 + tid] = sn;
                rc[kJacMax + tid] = npp;
                rc[3 * (kJacMax / 2) + tid] = nqq;
                pp[2 * np + tid] = act;
            }
            __syncthreads();
            // rows: J^T A
            for (int idx = tid; idx < np * k; idx += kJacThreads) {
                const int i = idx / k, col = idx % k;
                const int p = pp[i], q = pp[np + i];
                const double sn = rc[kJacMax / 2 + i];
                if (pp[2 * np + i]) {
                    const double c = rc[i], ap = a[p][col], aq = a[q][col];
                    a[p][col] = c * ap - sn * aq;
                    a[q][col] = sn * ap + c * aq;
                }
            }
            __syncthreads();
            // columns: (J^T A) J and V J
            for (int idx = tid; idx < np * k; idx += kJacThreads) {
                const int i = idx / k, r = idx % k;
                const int p = pp[i], q = pp[np + i];
                const double sn = rc[kJacMax / 2 + i];
                if (pp[2 * np + i]) {
                    const double c = rc[i];
                    const double ap = a[r][p], aq = a[r][q];
                    a[r][p] = c * ap - sn * aq;
                    a[r][q] = sn * ap + c * aq;
                    const double vp = v[r][p], vq = v[r][q];
                    v[r][p] = c * vp - sn * vq;
                    v[r][q] = sn * vp + c * vq;
                }
            }
            __syncthreads();
            // the rotated 2x2 block exactly as the reference writes it
            if (tid < np) {
                const int p = pp[tid], q = pp[np + tid];
                if (pp[2 * np + tid]) {
                    a[p][p] = rc[kJacMax + tid];
                    a[q][q] = rc[3 * (kJacMax / 2) + tid];
                    a[p][q] = 0.0;
                    a[q][p] = 0.0;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        // stable ascending order of the diagonal (np.argsort kind="stable")
        for (int i = 0; i < k; ++i) order[i] = i;
        for (int i = 1; i < k; ++i) {
            int oi = order[i];
            double key = a[oi][oi];
            int j = i - 1;
            while (j >= 0 && a[order[j]][order[j]] > key) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = oi;
        }
        info[0] = sweep;
    }
    __syncthreads();
    for (int i = tid; i < k; i += kJacThreads) evals[i] = a[order[i]][order[i]];
    for (int idx = tid; idx < k * k; idx += kJacThreads) {
        int r = idx / k, cidx = idx % k;
        evecs[r * k + cidx] = v[r][order[cidx]];
    }
}

// ---------------------------------------------------------------------------
// Register-streaming passes (16-byte aligned operands, K <= 32).  A thread owns
// element pairs (128-bit loads) and walks all k vectors of the pair itself, so
// no cross-warp reduction or barrier sits inside the stream and each thread
// keeps up to 2k independent loads in flight.  The dot-product phase re-reads
// the k V pairs the same thread just loaded (L2 hits: only the first touch
// costs HBM).  Per-thread accumulators are reduced once at the end.
constexpr int kRegBlock = 256;
// roots handled by the register residual pass (more roots keep the TMA-staged pass)
constexpr int kRegMaxRoots = 4;

// Per-block partials: vector slots [0, KV) (thread-owned subsets, see below)
// followed by NX scalar accumulators.  With S threads per element pair, thread
// h = lane % S owns vectors i = h + S j (j < K/S); a lane-strided shuffle tree
// reduces each subset among its own lanes only.
template <int K, int S, int NX>
__device__ __forceinline__ void block_store_partials(const double (&acc)[K / S], const double (&xs)[NX],
                                                     double *__restrict__ partial, int stride) {
    __shared__ double red[kRegBlock / 32][K + NX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane % S;
#pragma unroll
    for (int j = 0; j < K / S; ++j) {
        double v = acc[j];
#pragma unroll
        for (int o = 16; o >= S; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane < S) red[warp][h + S * j] = v;
    }
#pragma unroll
    for (int j = 0; j < NX; ++j) {
        const double v = warp_sum(xs[j]);
        if (lane == 0) red[warp][K + j] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K + NX; i += blockDim.x) {
        double sum = 0.0;
        for (int w = 0; w < kRegBlock / 32; ++w) sum += red[w][i];
        partial[(i64)blockIdx.x * stride + i] = sum;
    }
}

template <int S>
__device__ __forceinline__ double2 pair_sum(double2 v) {  // sum over the S lanes sharing an element pair
    if (S > 1) {  // only the S lanes of the group take part: other groups may have left the loop
        const unsigned gm = ((1u << S) - 1u) << ((threadIdx.x & 31) & ~(unsigned)(S - 1));
#pragma unroll
        for (int o = 1; o < S; o <<= 1) {
            v.x += __shfl_xor_sync(gm, v.x, o);
            v.y += __shfl_xor_sync(gm, v.y, o);
        }
    }
    return v;
}

// Lane 0 of each warp bulk-prefetches, into L2, the element pairs the warp
// touches in vector v this iteration, so the thread's register-staged loads
// (8 vectors at a time) find them in L2 instead of paying one HBM latency per
// group of 8.
__device__ __forceinline__ void warp_prefetch(const double *v, i64 p_warp, i64 np, int npairs) {
    if (p_warp < np) {
        const i64 cnt = min((i64)npairs, np - p_warp);
        prefetch_l2(v + 2 * p_warp, (uint32_t)(cnt * 16));
    }
}

__device__ __forceinline__ double precond_div(double r, double d, double th, double delta) {
    const double g = d - th;
    return r / ((g >= 0.0 ? 1.0 : -1.0) * fmax(fabs(g), delta));
}

// Residuals, preconditioned corrections and V^T t_jp (davidson.py:252-258,159-163).
// partial per block (stride K+1+M): [0,K) dots | K: |t_jp|^2 | K+1+j: |r_j|^2
// S threads per element pair (S = 2 halves the per-thread accumulators at K = 32).
template <int K, int M, int S>
__global__ void __launch_bounds__(kRegBlock, 2)
residual_reg(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
             const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
             const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
             double *__restrict__ partial, int pf) {
    constexpr int KS = K / S;
    __shared__ double ys[K * M];
    __shared__ double th[M];
    for (int idx = threadIdx.x; idx < K * M; idx += blockDim.x) {
        const int i = idx / M, j = idx % M;
        ys[idx] = (i < k && j < m) ? Y[i * m + j] : 0.0;
    }
    if (threadIdx.x < M) th[threadIdx.x] = threadIdx.x < m ? theta[threadIdx.x] : 0.0;
    __syncthreads();
    const int h = (threadIdx.x & 31) % S;
    double acc[KS], xs[1 + M];
#pragma unroll
    for (int i = 0; i < KS; ++i) acc[i] = 0.0;
#pragma unroll
    for (int j = 0; j <= M; ++j) xs[j] = 0.0;
    const i64 np = n / 2, stride = (i64)gridDim.x * blockDim.x / S;
    for (i64 p = ((i64)blockIdx.x * blockDim.x + threadIdx.x) / S; p < np; p += stride) {
        if (pf && (threadIdx.x & 31) == 0) {
            for (int i = 0; i < k; ++i) {
                warp_prefetch(V + i * ldv, p, np, 32 / S);
                warp_prefetch(W + i * ldv, p, np, 32 / S);
            }
            warp_prefetch(diag, p, np, 32 / S);
        }
        double2 u[M], wy[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = wy[j] = make_double2(0.0, 0.0);
#pragma unroll
        for (int q0 = 0; q0 < KS; q0 += 4) {  // 4 vectors x (V, W): 8 independent loads, then the FMAs
            double2 v[4], w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = h + S * (q0 + e);
                const bool on = q0 + e < KS && i < k;
                v[e] = on ? reinterpret_cast<const double2 *>(V + i * ldv)[p] : make_double2(0.0, 0.0);
                w[e] = on ? __ldcs(reinterpret_cast<const double2 *>(W + i * ldv) + p) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = h + S * (q0 + e);
                if (q0 + e < KS && i < k) {
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        const double y = ys[i * M + j];
                        u[j].x = fma(y, v[e].x, u[j].x);
                        u[j].y = fma(y, v[e].y, u[j].y);
                        wy[j].x = fma(y, w[e].x, wy[j].x);
                        wy[j].y = fma(y, w[e].y, wy[j].y);
                    }
                }
            }
        }
        const double2 d = __ldcs(reinterpret_cast<const double2 *>(diag) + p);
        double2 tj = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if (j < m) {
                u[j] = pair_sum<S>(u[j]);
                wy[j] = pair_sum<S>(wy[j]);
                const double rx = wy[j].x - th[j] * u[j].x, ry = wy[j].y - th[j] * u[j].y;
                const double2 t = make_double2(precond_div(rx, d.x, th[j], delta), precond_div(ry, d.y, th[j], delta));
                if (h == 0) {
                    __stcs(reinterpret_cast<double2 *>(T + j * ldt) + p, t);
                    xs[1 + j] = fma(rx, rx, fma(ry, ry, xs[1 + j]));
                }
                if (j == jp) tj = t;
            }
        }
        if (h == 0) xs[0] = fma(tj.x, tj.x, fma(tj.y, tj.y, xs[0]));
#pragma unroll
        for (int q = 0; q < KS; ++q) {
            const int i = h + S * q;
            if (i < k) {
                const double2 v = __ldcs(reinterpret_cast<const double2 *>(V + i * ldv) + p);
                acc[q] = fma(v.x, tj.x, fma(v.y, tj.y, acc[q]));
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x < S) {  // odd tail element: the S lanes of pair 0
        const i64 e = n - 1;
        double u[M], wy[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = wy[j] = 0.0;
        for (int i = 0; i < k; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
                u[j] = fma(ys[i * M + j], V[i * ldv + e], u[j]);
                wy[j] = fma(ys[i * M + j], W[i * ldv + e], wy[j]);
            }
        double tj = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j)
            if (j < m) {
                const double r = wy[j] - th[j] * u[j];
                const double t = precond_div(r, diag[e], th[j], delta);
                if (h == 0) {
                    T[j * ldt + e] = t;
                    xs[1 + j] = fma(r, r, xs[1 + j]);
                }
                if (j == jp) tj = t;
            }
        if (h == 0) xs[0] = fma(tj, tj, xs[0]);
#pragma unroll
        for (int q = 0; q < KS; ++q)
            if (h + S * q < k) acc[q] = fma(V[(h + S * q) * ldv + e], tj, acc[q]);
    }
    block_store_partials<K, S, 1 + M>(acc, xs, partial, K + 1 + M);
}

// Residual pass streamed through shared memory (the default for k <= 32, m <= 4).
// One CTA per SM walks tiles of TT elements (256; 192 for K = 32).  A producer warp
// bulk-copies (cp.async.bulk, the copies spread over its lanes) each tile's 2k+1 slices (k V,
// k W, diag) into one of NS stages, NS sized so the stages hold ~210 KB (k = 5: 8 stages of
// 22 KB; k = 16: 3 of 66 KB; k = 24-32: 2 of ~100 KB), i.e. NS-1 tiles in flight per SM
// while the consumers compute one.  Consumers take one element per thread, release a stage
// per warp on its `empty` mbarrier (no CTA-wide barrier per tile), and read the V^T t_jp
// projections' V from the stage instead of re-reading it.
// Measured per k at 1e8 elements against the register pass it replaced (profiles/r4j, r4k):
// k = 4: 5.1 vs 4.7 TB/s, k = 8-24: 6.7-7.0 vs 4.2-6.3, k = 25-28: 6.2-6.6 vs 5.9-6.1,
// k = 32: 6.1 vs 6.3; three roots k = 24/32: 6.4/5.9 vs 4.0/3.3.  A single issuing lane
// (instead of the warp) made it clock-sensitive: 5.3-6.7 TB/s at k = 8 from box to box.
// partial per block (stride K+1+M): [0,K) dots | K: |t_jp|^2 | K+1+j: |r_j|^2
// elements per tile = consumer threads: 256, or 192 for K = 32 so that two stages of
// 65 slices (97.5 KB each) fit in shared memory
__host__ __device__ constexpr int res_stream_tile(int K) { return K <= 24 ? 256 : 192; }
constexpr int kResMaxStages = 8;
constexpr int kResStreamMaxK = 32;
constexpr int kResStreamTile = 256;  // vdots2_stream's tile
constexpr size_t kResStageBudget = 210 * 1024;

inline int res_stream_stages(int K, int k) {
    const size_t stage = sizeof(double) * (size_t)(2 * k + 1) * res_stream_tile(K);
    return (int)std::max<size_t>(2, std::min<size_t>(kResMaxStages, kResStageBudget / stage));
}
inline size_t res_stream_smem(int K, int k) {
    return 256 + sizeof(double) * (size_t)res_stream_stages(K, k) * (size_t)(2 * k + 1) * res_stream_tile(K);
}

template <int NCONS>
__device__ __forceinline__ void consumers_sync() {  // named barrier 1 over the consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(NCONS) : "memory");
}

template <int K, int M>
__global__ void __launch_bounds__(res_stream_tile(K) + 32, 1)
residual_stream(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
                const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
                const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
                double *__restrict__ partial, int ns) {
    constexpr int TT = res_stream_tile(K), NW = TT / 32;  // + one producer warp
    extern __shared__ __align__(128) unsigned char rss[];
    uint64_t *full = reinterpret_cast<uint64_t *>(rss), *empty = full + kResMaxStages;
    double *stage0 = reinterpret_cast<double *>(rss + 256);
    __shared__ double ys[K * M];
    __shared__ double th[M];
    __shared__ double red[NW][K + 1 + M];
    const i64 sstride = (i64)(2 * k + 1) * TT;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int idx = t; idx < K * M; idx += blockDim.x) {
        const int i = idx / M, j = idx % M;
        ys[idx] = (i < k && j < m) ? Y[i * m + j] : 0.0;
    }
    if (t < M) th[t] = t < m ? theta[t] : 0.0;
    if (t == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const i64 ntiles = (n + TT - 1) / TT;
    if (warp == NW) {  // producer warp: lane 0 arms the stage, the lanes issue its 2k+1 copies
        int it = 0;
        for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it % ns;
            if (it >= ns) mbar_wait(&empty[s], (uint32_t)(((it / ns) - 1) & 1));
            const i64 base = tile * TT, cnt = min((i64)TT, n - base);
            const uint32_t b = bulk_bytes(cnt);
            double *st = stage0 + s * sstride;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], b * (uint32_t)(2 * k + 1));
            __syncwarp();
            if (b) {
                for (int c = lane; c <= 2 * k; c += 32) {  // slice c: V_c, W_(c-k), diag
                    const double *src = c < k ? V + c * ldv : (c < 2 * k ? W + (c - k) * ldv : diag);
                    tma_load_1d(st + (i64)c * TT, src + base, b, &full[s]);
                }
            }
        }
        return;
    }
    const int e = t;
    double acc[K], rn2[M], tn2 = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = 0.0;
    int it = 0;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % ns;
        const i64 base = tile * TT, cnt = min((i64)TT, n - base);
        double *st = stage0 + s * sstride;
        mbar_wait(&full[s], (uint32_t)((it / ns) & 1));
        if (cnt & 1) {  // odd last element: plain loads (bulk copies move 16-byte multiples)
            if (t == 0) {
                const i64 q = cnt - 1;
                for (int i = 0; i < k; ++i) {
                    st[(i64)i * TT + q] = V[i * ldv + base + q];
                    st[(i64)(k + i) * TT + q] = W[i * ldv + base + q];
                }
                st[(i64)(2 * k) * TT + q] = diag[base + q];
                fence_proxy_async_smem();  // before the stage can be refilled by bulk copies
            }
            consumers_sync<TT>();
        }
        double u[M], wy[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = wy[j] = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (i < k) {
                const double v = st[(i64)i * TT + e], w = st[(i64)(k + i) * TT + e];
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const double y = ys[i * M + j];
                    u[j] = fma(y, v, u[j]);
                    wy[j] = fma(y, w, wy[j]);
                }
            }
        }
        if (e < cnt) {
            const double d = st[(i64)(2 * k) * TT + e];
            double tj = 0.0;
#pragma unroll
            for (int j = 0; j < M; ++j) {
                if (j < m) {
                    const double r = wy[j] - th[j] * u[j];
                    const double tv = precond_div(r, d, th[j], delta);
                    __stcs(T + j * ldt + base + e, tv);
                    rn2[j] = fma(r, r, rn2[j]);
                    if (j == jp) tj = tv;
                }
            }
            tn2 = fma(tj, tj, tn2);
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i < k) acc[i] = fma(st[(i64)i * TT + e], tj, acc[i]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }
    // block reduction over the consumer warps
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const double v = warp_sum(acc[i]);
        if (lane == 0) red[warp][i] = v;
    }
    tn2 = warp_sum(tn2);
#pragma unroll
    for (int j = 0; j < M; ++j) rn2[j] = warp_sum(rn2[j]);
    if (lane == 0) {
        red[warp][K] = tn2;
#pragma unroll
        for (int j = 0; j < M; ++j) red[warp][K + 1 + j] = rn2[j];
    }
    consumers_sync<TT>();
    for (int i = t; i < K + 1 + M; i += TT) {
        double sum = 0.0;
        for (int w = 0; w < NW; ++w) sum += red[w][i];
        partial[(i64)blockIdx.x * (K + 1 + M) + i] = (i < K && i >= k) ? 0.0 : sum;
    }
}

// V^T w and V^T u (the T column and the Gram row) streamed like residual_stream: a producer
// warp bulk-copies each 256-element tile's k + 2 slices (k V, w, u) into stages sized to
// ~210 KB; 8 consumer warps, one element per thread, 2k accumulators per thread.
// partial per block (stride 2K): [0,K) V^T w | [K,2K) V^T u
template <int K>
__global__ void __launch_bounds__(kResStreamTile + 32, 1)
vdots2_stream(const double *__restrict__ V, int k, i64 ldv, i64 n, const double *__restrict__ w,
              const double *__restrict__ u, double *__restrict__ partial, int ns) {
    constexpr int TT = kResStreamTile, NW = TT / 32;
    extern __shared__ __align__(128) unsigned char vss[];
    uint64_t *full = reinterpret_cast<uint64_t *>(vss), *empty = full + kResMaxStages;
    double *stage0 = reinterpret_cast<double *>(vss + 256);
    __shared__ double red[NW][2 * K];
    const i64 sstride = (i64)(k + 2) * TT;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const i64 ntiles = (n + TT - 1) / TT;
    if (warp == NW) {  // producer warp
        int it = 0;
        for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it % ns;
            if (it >= ns) mbar_wait(&empty[s], (uint32_t)(((it / ns) - 1) & 1));
            const i64 base = tile * TT, cnt = min((i64)TT, n - base);
            const uint32_t b = bulk_bytes(cnt);
            double *st = stage0 + s * sstride;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], b * (uint32_t)(k + 2));
            __syncwarp();
            if (b) {
                for (int c = lane; c < k + 2; c += 32) {  // slice c: V_c, w, u
                    const double *src = c < k ? V + c * ldv : (c == k ? w : u);
                    tma_load_1d(st + (i64)c * TT, src + base, b, &full[s]);
                }
            }
        }
        return;
    }
    double aw[K], au[K];
#pragma unroll
    for (int i = 0; i < K; ++i) aw[i] = au[i] = 0.0;
    int it = 0;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % ns;
        const i64 base = tile * TT, cnt = min((i64)TT, n - base);
        double *st = stage0 + s * sstride;
        mbar_wait(&full[s], (uint32_t)((it / ns) & 1));
        if (cnt & 1) {  // odd last element: plain loads
            if (t == 0) {
                const i64 q = cnt - 1;
                for (int i = 0; i < k; ++i) st[(i64)i * TT + q] = V[i * ldv + base + q];
                st[(i64)k * TT + q] = w[base + q];
                st[(i64)(k + 1) * TT + q] = u[base + q];
                fence_proxy_async_smem();
            }
            consumers_sync<TT>();
        }
        if (t < cnt) {
            const double we = st[(i64)k * TT + t], ue = st[(i64)(k + 1) * TT + t];
#pragma unroll
            for (int i = 0; i < K; ++i) {
                if (i < k) {
                    const double v = st[(i64)i * TT + t];
                    aw[i] = fma(v, we, aw[i]);
                    au[i] = fma(v, ue, au[i]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const double a = warp_sum(aw[i]), b = warp_sum(au[i]);
        if (lane == 0) {
            red[warp][i] = a;
            red[warp][K + i] = b;
        }
    }
    consumers_sync<TT>();
    for (int i = t; i < 2 * K; i += TT) {
        double sum = 0.0;
        for (int ww = 0; ww < NW; ++ww) sum += red[ww][i];
        partial[(i64)blockIdx.x * 2 * K + i] = (i % K) < k ? sum : 0.0;
    }
}

inline int vdots2_stream_stages(int k) {
    const size_t stage = sizeof(double) * (size_t)(k + 2) * kResStreamTile;
    return (int)std::max<size_t>(2, std::min<size_t>(kResMaxStages, kResStageBudget / stage));
}

// t_new = t - V c ; out = scale * t_new (out may alias t) ; dots V_i . t_new (i < kdot) ; |t_new|^2
// partial per block (stride K+1): [0,K) dots | K: |t_new|^2 ; S threads per element pair.
template <int K, bool DOTS, int S>
__global__ void __launch_bounds__(kRegBlock, 2)
gs_reg(const double *__restrict__ V, int k, i64 ldv, i64 n, const double *__restrict__ c, int kdot, const double *t,
       double *out, const double *__restrict__ scale, double *__restrict__ partial, int pf) {
    constexpr int KS = K / S;
    __shared__ double cs[K];
    for (int i = threadIdx.x; i < K; i += blockDim.x) cs[i] = i < k ? c[i] : 0.0;
    __syncthreads();
    const double sc = scale ? *scale : 1.0;
    const int h = (threadIdx.x & 31) % S;
    double acc[KS], xs[1] = {0.0};
#pragma unroll
    for (int i = 0; i < KS; ++i) acc[i] = 0.0;
    const i64 np = n / 2, stride = (i64)gridDim.x * blockDim.x / S;
    for (i64 p = ((i64)blockIdx.x * blockDim.x + threadIdx.x) / S; p < np; p += stride) {
        if (pf && (threadIdx.x & 31) == 0) {
            for (int i = 0; i < k; ++i) warp_prefetch(V + i * ldv, p, np, 32 / S);
            warp_prefetch(t, p, np, 32 / S);
        }
        double2 sv = make_double2(0.0, 0.0);
#pragma unroll
        for (int q0 = 0; q0 < KS; q0 += 8) {  // 8 independent loads ahead of each FMA chain
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = h + S * (q0 + u);
                if (q0 + u < KS && i < k)
                    v[u] = DOTS ? reinterpret_cast<const double2 *>(V + i * ldv)[p]
                                : __ldcs(reinterpret_cast<const double2 *>(V + i * ldv) + p);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = h + S * (q0 + u);
                if (q0 + u < KS && i < k) {
                    sv.x = fma(cs[i], v[u].x, sv.x);
                    sv.y = fma(cs[i], v[u].y, sv.y);
                }
            }
        }
        sv = pair_sum<S>(sv);
        const double2 t0 = reinterpret_cast<const double2 *>(t)[p];
        const double2 tv = make_double2(t0.x - sv.x, t0.y - sv.y);
        if (h == 0) {
            __stcs(reinterpret_cast<double2 *>(out) + p, make_double2(tv.x * sc, tv.y * sc));  // no dirty-L2 backlog
            xs[0] = fma(tv.x, tv.x, fma(tv.y, tv.y, xs[0]));
        }
        if (DOTS) {
#pragma unroll
            for (int q = 0; q < KS; ++q) {
                const int i = h + S * q;
                if (i < kdot) {
                    const double2 v = __ldcs(reinterpret_cast<const double2 *>(V + i * ldv) + p);  // L2 hit
                    acc[q] = fma(v.x, tv.x, fma(v.y, tv.y, acc[q]));
                }
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x < S) {
        const i64 e = n - 1;
        double sx = 0.0;
        for (int i = 0; i < k; ++i) sx = fma(cs[i], V[i * ldv + e], sx);
        const double x = t[e] - sx;
        if (h == 0) {
            out[e] = x * sc;
            xs[0] = fma(x, x, xs[0]);
        }
#pragma unroll
        for (int q = 0; q < KS; ++q)
            if (h + S * q < kdot) acc[q] = fma(V[(h + S * q) * ldv + e], x, acc[q]);
    }
    block_store_partials<K, S, 1>(acc, xs, partial, K + 1);
}

// out[j] <- sum_i Y[i, j] V[i] for j < nout <= 8: the thick restart in place
// (out = V, davidson.py:280-289) and the final Ritz vectors (out = U,
// davidson.py:256).  Thread per element pair; the whole pair column of V is
// read (L2-prefetched in bulk, then 8 vectors at a time) before any output is
// written, so the in-place form is safe.
template <int K>
__global__ void __launch_bounds__(kRegBlock, 2)
mix_reg(const double *V, int k, i64 ldv, i64 n, const double *__restrict__ Y, int nout, double *out, i64 ldo) {
    __shared__ double ys[K * 8];
    for (int idx = threadIdx.x; idx < K * 8; idx += blockDim.x) {
        const int i = idx / 8, j = idx % 8;
        ys[idx] = (i < k && j < nout) ? Y[i * nout + j] : 0.0;
    }
    __syncthreads();
    const i64 np = n / 2, stride = (i64)gridDim.x * blockDim.x;
    for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += stride) {
        if ((threadIdx.x & 31) == 0)
            for (int i = 0; i < k; ++i) warp_prefetch(V + i * ldv, p, np, 32);
        double2 u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = make_double2(0.0, 0.0);
#pragma unroll
        for (int i0 = 0; i0 < K; i0 += 8) {
            double2 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (i0 + q < k) v[q] = __ldcs(reinterpret_cast<const double2 *>(V + (i0 + q) * ldv) + p);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (i0 + q < k)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const double y = ys[(i0 + q) * 8 + j];
                        u[j].x = fma(y, v[q].x, u[j].x);
                        u[j].y = fma(y, v[q].y, u[j].y);
                    }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < nout) reinterpret_cast<double2 *>(out + j * ldo)[p] = u[j];
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const i64 e = n - 1;
        double u[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < k; ++i) {
            const double v = V[i * ldv + e];
#pragma unroll
            for (int j = 0; j < 8; ++j) u[j] = fma(ys[i * 8 + j], v, u[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < nout) out[j * ldo + e] = u[j];
    }
}

inline bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline bool vec_ok(const double *V, i64 ldv) { return al16(V) && ldv % 2 == 0; }
template <class... P>
inline bool vec_ok(const double *V, i64 ldv, const double *p, P... rest) {
    return al16(p) && vec_ok(V, ldv, rest...);
}

// Pass variants (read per launch, so tests can select each one in-process; tests/test_gpu_kernels.py):
//   default      k <= 32: register passes (residual_reg, gs_reg, mix_reg); k > 32: TMA-staged passes
//   SBD_DAV_TMA=1  TMA-staged passes for every k
//   SBD_NO_TMA=1   no TMA: tile / generic passes
inline bool use_tma() {
    const char *e = getenv("SBD_NO_TMA");
    return !(e && *e && *e != '0');
}

inline bool use_reg() {
    const char *e = getenv("SBD_DAV_TMA");
    return !(e && *e == '1');
}

inline bool use_res_stream() {  // SBD_RES_STREAM=0: the register-staged residual pass (A/B, tests)
    const char *e = getenv("SBD_RES_STREAM");
    return !(e && *e == '0');
}

// lanes per element pair for pass `which` (0 residual, 1 CGS); SBD_RES_SPLIT / SBD_GS_SPLIT
// override the default for A/B measurements
inline int split_lanes(int which, int dflt) {
    const char *e = getenv(which == 0 ? "SBD_RES_SPLIT" : "SBD_GS_SPLIT");
    const int v = e && *e ? atoi(e) : dflt;
    return (v == 1 || v == 2 || v == 4) ? v : dflt;
}

int tile_blocks(sbd_ctx *ctx, i64 n, int tt) {
    i64 b = (n + tt - 1) / tt;
    return (int)std::max<i64>(1, std::min<i64>(b, (i64)ctx->num_sms * 8));
}

int red_blocks(sbd_ctx *ctx, i64 n) {
    i64 b = (n + kBlock - 1) / kBlock;
    return (int)std::max<i64>(1, std::min<i64>(b, (i64)ctx->num_sms * 4));
}

int ensure_red(sbd_ctx *ctx, int nblocks, int stride) {
    nblocks = std::max(nblocks, ctx->num_sms * 8);
    SBD_CUDA(ctx, ctx->red.ensure(sizeof(double) * (size_t)nblocks * stride + 64));
    return SBD_OK;
}

int check_k(sbd_ctx *ctx, int k) {
    if (k < 0 || k > 64) return sbd_fail(ctx, SBD_EINVAL, "subspace size must be in [0, 64]");
    return SBD_OK;
}

template <template <int> class Launch, class... Args>
int dispatch_k(int k, Args... args) {
    if (k <= 8) return Launch<8>::run(args...);
    if (k <= 16) return Launch<16>::run(args...);
    if (k <= 24) return Launch<24>::run(args...);
    if (k <= 32) return Launch<32>::run(args...);
    return Launch<64>::run(args...);
}

template <int K>
struct VdotsL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *w, double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, K)) return rc;
        if (vec_ok(V, ldv, w)) vdots_kernel<K, true><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, ctx->red.as<double>());
        else vdots_kernel<K, false><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, ctx->red.as<double>());
        finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nb, K, k, K, k, out);
        SBD_LAUNCHED(ctx, "vdots");
        return SBD_OK;
    }
};

template <int K>
struct Vdots2L {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *w, const double *u,
                   double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, 2 * K)) return rc;
        if (K <= 32 && vec_ok(V, ldv, w, u) && use_reg() && use_res_stream()) {
            constexpr int KS = K <= 32 ? K : 32;
            const int ns = vdots2_stream_stages(k);
            const size_t smem = 256 + sizeof(double) * (size_t)ns * (size_t)(k + 2) * kResStreamTile;
            const int nt = (int)std::max<i64>(1, std::min<i64>((n + kResStreamTile - 1) / kResStreamTile,
                                                               ctx->num_sms));
            (void)sbd_smem_attr((const void *)vdots2_stream<KS>, ctx->device, smem);  // launch errors surface below
            vdots2_stream<KS><<<nt, kResStreamTile + 32, smem, ctx->stream>>>(V, k, ldv, n, w, u,
                                                                                ctx->red.as<double>(), ns);
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nt, 2 * K, k, K, k, out);
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>() + K, nt, 2 * K, k, K, k, out + k);
            SBD_LAUNCHED(ctx, "vdots2");
            return SBD_OK;
        }
        if (vec_ok(V, ldv, w, u)) {
            const int nt = tile_blocks(ctx, n, 1024);
            vdots2_tile<K><<<nt, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, u, ctx->red.as<double>());
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nt, 2 * K, k, K, k, out);
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>() + K, nt, 2 * K, k, K, k, out + k);
            SBD_LAUNCHED(ctx, "vdots2");
            return SBD_OK;
        }
        vdots2_kernel<K, false><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, u, ctx->red.as<double>());
        finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nb, 2 * K, k, K, k, out);
        finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>() + K, nb, 2 * K, k, K, k, out + k);
        SBD_LAUNCHED(ctx, "vdots2");
        return SBD_OK;
    }
};

template <int K>
struct ResidL {
    // returns (blocks, partial stride) of the launched kernel
    template <int M>
    static std::pair<int, int> launch(sbd_ctx *ctx, int nb, const double *V, const double *W, int k, i64 ldv, i64 n,
                                      const double *Y, const double *theta, int m, int jp, const double *diag,
                                      double delta, double *T, i64 ldt) {
        if (K <= kResStreamMaxK && M <= kRegMaxRoots && vec_ok(V, ldv, W, diag, T) &&
            ldt % 2 == 0 && use_reg() && use_res_stream()) {
            constexpr int KS = K <= kResStreamMaxK ? K : kResStreamMaxK;
            constexpr int TT = res_stream_tile(KS);
            const size_t smem = res_stream_smem(KS, k);
            const int nt = (int)std::max<i64>(1, std::min<i64>((n + TT - 1) / TT, ctx->num_sms));
            (void)sbd_smem_attr((const void *)residual_stream<KS, M>, ctx->device, smem);  // launch errors surface below
            residual_stream<KS, M><<<nt, TT + 32, smem, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag,
                                                                      delta, T, ldt, ctx->red.as<double>(),
                                                                      res_stream_stages(KS, k));
            return {nt, K + 1 + M};
        }
        if (K <= 32 && M <= kRegMaxRoots && vec_ok(V, ldv, W, diag, T) && ldt % 2 == 0 && use_reg()) {
            const int nt = ctx->num_sms * 2;
            constexpr int KR = K <= 32 ? K : 32;
            // S lanes per element pair split the k vectors: fewer accumulators per thread, so the
            // compiler keeps the loads of a thread in flight together (k > 16)
            const int sp = split_lanes(0, KR >= 24 ? 2 : 1);
            // L2 bulk prefetch of the residual's 2k+1 slices: measured slower once the loads are
            // batched (the bulk-prefetch issue rate becomes the limit); SBD_RES_PF=1 re-enables it
            const char *pfe = getenv("SBD_RES_PF");
            const int pf = pfe && *pfe == '1' ? 1 : 0;
            if (sp == 4)
                residual_reg<KR, M, 4><<<nt, kRegBlock, 0, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag,
                                                                         delta, T, ldt, ctx->red.as<double>(), pf);
            else if (sp == 2)
                residual_reg<KR, M, 2><<<nt, kRegBlock, 0, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag,
                                                                         delta, T, ldt, ctx->red.as<double>(), pf);
            else
                residual_reg<KR, M, 1><<<nt, kRegBlock, 0, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag,
                                                                         delta, T, ldt, ctx->red.as<double>(), pf);
            return {nt, K + 1 + M};
        }
        const int TTA = tma_tile(2 * k + 1);
        const size_t smem_tma = 128 + sizeof(double) * (2 * (size_t)(2 * k + 1) * TTA + TTA + 2 * 8 * M * (size_t)TTA);
        if (vec_ok(V, ldv, W, diag, T) && ldt % 2 == 0 && use_tma() && smem_tma <= 220 * 1024 &&
            TTA <= 32 * resid_epl(K)) {
            const size_t smem = smem_tma;
            const int nt = std::max(1, std::min<int>((int)((n + TTA - 1) / TTA), ctx->num_sms));
            (void)sbd_smem_attr((const void *)residual_tma<K, M>, ctx->device, 220 * 1024);  // launch errors surface below
            residual_tma<K, M><<<nt, kBlock, smem, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T,
                                                                 ldt, ctx->red.as<double>());
            return {nt, K + 1 + M};
        }
        if (vec_ok(V, ldv, W, diag, T) && ldt % 2 == 0) {
            constexpr int TT = 512 / M;
            const int nt = tile_blocks(ctx, n, TT);
            const size_t smem = sizeof(double2) * (2 * kWarpsT * M * (TT / 2) + TT / 2);
            (void)sbd_smem_attr((const void *)residual_tile<K, M>, ctx->device, smem);  // launch errors surface below
            residual_tile<K, M><<<nt, kBlock, smem, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T,
                                                                  ldt, ctx->red.as<double>());
            return {nt, K + 1 + M};
        }
        residual_kernel<K, M, false><<<nb, kBlock, 0, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T,
                                                                    ldt, ctx->red.as<double>());
        return {nb, K + 1 + M};
    }
    static int run(sbd_ctx *ctx, const double *V, const double *W, int k, i64 ldv, i64 n, const double *Y,
                   const double *theta, int m, int jp, const double *diag, double delta, double *T, i64 ldt,
                   double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, (int)ctx->num_sms * 8, K + 9)) return rc;
        std::pair<int, int> bs;
        if (m == 1) bs = launch<1>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else if (m == 2) bs = launch<2>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else if (m <= 4) bs = launch<4>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else bs = launch<8>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), bs.first, bs.second, k, K, k + 1 + m, out);
        SBD_LAUNCHED(ctx, "residual_precond");
        return SBD_OK;
    }
};

template <int K>
struct GsL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *c, int kdot, double *t,
                   double *out, double *out_vec = nullptr, const double *scale = nullptr) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, K + 1)) return rc;
        double *dst = out_vec ? out_vec : t;
        if (K <= 32 && vec_ok(V, ldv, t) && al16(dst) && use_reg()) {
            const int nt = ctx->num_sms * 2;
            constexpr int KR = K <= 32 ? K : 32;
            const bool split = KR == 32 && split_lanes(1, 1) == 2;
            // L2 bulk prefetch helps the pass with the dot phase (it re-reads V), not the plain update;
            // SBD_GS_PF=0/1 forces it off/on
            const char *pfe = getenv("SBD_GS_PF");
            const int pf = pfe && *pfe ? (*pfe == '1') : (kdot > 0 ? 1 : 0);
            if (kdot > 0 && split)
                gs_reg<KR, true, 2><<<nt, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, dst, scale,
                                                                      ctx->red.as<double>(), pf);
            else if (kdot > 0)
                gs_reg<KR, true, 1><<<nt, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, dst, scale,
                                                                      ctx->red.as<double>(), pf);
            else if (split)
                gs_reg<KR, false, 2><<<nt, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, dst, scale,
                                                                       ctx->red.as<double>(), pf);
            else
                gs_reg<KR, false, 1><<<nt, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, dst, scale,
                                                                       ctx->red.as<double>(), pf);
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nt, K + 1, kdot, K, kdot + 1, out);
            SBD_LAUNCHED(ctx, "gs_update");
            return SBD_OK;
        }
        if (vec_ok(V, ldv, t) && use_tma()) {
            const int TTA = tma_tile(k + 1);
            const size_t smem = 128 + sizeof(double) * 2 * (size_t)(k + 1) * TTA;
            const int nt = std::max(1, std::min<int>((int)((n + TTA - 1) / TTA), ctx->num_sms));
            SBD_CUDA(ctx, sbd_smem_attr((const void *)gs_tma<K>, ctx->device, 220 * 1024));
            gs_tma<K><<<nt, kBlock, smem, ctx->stream>>>(V, k, ldv, n, c, kdot, t, dst, scale, ctx->red.as<double>());
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nt, K + 1, kdot, K, kdot + 1, out);
            SBD_LAUNCHED(ctx, "gs_update");
            return SBD_OK;
        }
        // non-TMA paths update t in place (the finalize form may clobber t), then scale into out_vec
        if (vec_ok(V, ldv, t)) {
            const int nt = tile_blocks(ctx, n, 512);
            gs_tile<K><<<nt, kBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, ctx->red.as<double>());
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nt, K + 1, kdot, K, kdot + 1, out);
        } else {
            gs_kernel<K, false><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, ctx->red.as<double>());
            finish_partials<<<kFinishBlocks, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nb, K + 1, kdot, K, kdot + 1, out);
        }
        if (out_vec) scale_copy_kernel<<<nb * 2, kBlock, 0, ctx->stream>>>(t, out_vec, n, scale);
        SBD_LAUNCHED(ctx, "gs_update");
        return SBD_OK;
    }
};

template <int K>
struct RotL {
    static int run(sbd_ctx *ctx, double *V, int k, i64 ldv, i64 n, const double *Y, int keep) {
        if (K <= 32 && keep <= 8 && vec_ok(V, ldv) && use_reg()) {
            mix_reg<(K <= 32 ? K : 32)><<<ctx->num_sms * 2, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, keep, V, ldv);
            SBD_LAUNCHED(ctx, "rotate");
            return SBD_OK;
        }
        rotate_kernel<K><<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, keep);
        SBD_LAUNCHED(ctx, "rotate");
        return SBD_OK;
    }
};

template <int K>
struct CombL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *Y, int m, double *U, i64 ldu) {
        if (K <= 32 && m <= 8 && vec_ok(V, ldv) && al16(U) && ldu % 2 == 0 && use_reg()) {
            mix_reg<(K <= 32 ? K : 32)><<<ctx->num_sms * 2, kRegBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, m, U, ldu);
            SBD_LAUNCHED(ctx, "combine");
            return SBD_OK;
        }
        combine_kernel<K><<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, m, U, ldu);
        SBD_LAUNCHED(ctx, "combine");
        return SBD_OK;
    }
};

}  // namespace

extern "C" {

int sbd_vdots(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *w, double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return SBD_OK;
    return dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, w, out);
}

int sbd_vdots2(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *w, const double *u,
               double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return SBD_OK;
    if (k > 32) {  // keep accumulators in registers: two single-RHS passes
        if (int rc = dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, w, out)) return rc;
        return dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, u, out + k);
    }
    return dispatch_k<Vdots2L>(k, ctx, V, k, (i64)ldv, (i64)n, w, u, out);
}

int sbd_residual_precond(sbd_ctx *ctx, const double *V, const double *W, int k, int64_t ldv, int64_t n,
                         const double *Y, const double *theta, int m, const double *diag, double delta, double *T,
                         int64_t ldt, double *rn2, double *proj) {
    // rn2/proj: single output buffer of k + 1 + m doubles laid out as
    // [V^T t_0 (k) | |t_0|^2 | |r_j|^2 (m)]; `rn2` must equal proj + k + 1.
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8 || m > k) return sbd_fail(ctx, SBD_EINVAL, "n_roots must be in [1, min(8, k)]");
    if (rn2 != proj + k + 1) return sbd_fail(ctx, SBD_EINVAL, "rn2 must alias proj + k + 1");
    return dispatch_k<ResidL>(k, ctx, V, W, k, (i64)ldv, (i64)n, Y, theta, m, 0, diag, delta, T, (i64)ldt, proj);
}

int sbd_residual_precond_target(sbd_ctx *ctx, const double *V, const double *W, int k, int64_t ldv, int64_t n,
                                const double *Y, const double *theta, int m, int target, const double *diag,
                                double delta, double *T, int64_t ldt, double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8 || m > k) return sbd_fail(ctx, SBD_EINVAL, "n_roots must be in [1, min(8, k)]");
    if (target < 0 || target >= m) return sbd_fail(ctx, SBD_EINVAL, "bad target root");
    return dispatch_k<ResidL>(k, ctx, V, W, k, (i64)ldv, (i64)n, Y, theta, m, target, diag, delta, T, (i64)ldt, out);
}

int sbd_gs_update(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *c, double *t,
                  double *out2) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return GsL<8>::run(ctx, V, 0, (i64)ldv, (i64)n, c, 0, t, out2);
    return dispatch_k<GsL>(k, ctx, V, k, (i64)ldv, (i64)n, c, k, t, out2, (double *)nullptr, (const double *)nullptr);
}

int sbd_gs_finalize(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *c, const double *t,
                    double *v_out, const double *scale, double *out_norm2) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return GsL<8>::run(ctx, V, 0, (i64)ldv, (i64)n, c, 0, const_cast<double *>(t), out_norm2, v_out, scale);
    return dispatch_k<GsL>(k, ctx, V, k, (i64)ldv, (i64)n, c, 0, const_cast<double *>(t), out_norm2, v_out, scale);
}

int sbd_gs_update_nodots(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *c, double *t,
                         double *out_norm2) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return GsL<8>::run(ctx, V, 0, (i64)ldv, (i64)n, c, 0, t, out_norm2);
    return dispatch_k<GsL>(k, ctx, V, k, (i64)ldv, (i64)n, c, 0, t, out_norm2, (double *)nullptr,
                           (const double *)nullptr);
}

int sbd_scale_copy(sbd_ctx *ctx, const double *src, double *dst, int64_t n, const double *scale) {
    SBD_CHECK_CTX(ctx);
    scale_copy_kernel<<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(src, dst, n, scale);
    SBD_LAUNCHED(ctx, "scale_copy");
    return SBD_OK;
}

int sbd_rotate(sbd_ctx *ctx, double *V, int k, int64_t ldv, int64_t n, const double *Y, int keep) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (keep < 1 || keep > k) return sbd_fail(ctx, SBD_EINVAL, "keep must be in [1, k]");
    return dispatch_k<RotL>(k, ctx, V, k, (i64)ldv, (i64)n, Y, keep);
}

int sbd_combine(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *Y, int m, double *U,
                int64_t ldu) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8) return sbd_fail(ctx, SBD_EINVAL, "m must be in [1, 8]");
    return dispatch_k<CombL>(k, ctx, V, k, (i64)ldv, (i64)n, Y, m, U, (i64)ldu);
}

int sbd_jacobi(sbd_ctx *ctx, const double *A, int k, int lda, double *evals, double *evecs, int max_sweeps,
               int *info) {
    SBD_CHECK_CTX(ctx);
    if (k < 1 || k > kJacMax) return sbd_fail(ctx, SBD_EINVAL, "jacobi size must be in [1, 64]");
    const int smem = (int)(sizeof(double) * (2 * kJacMax * (kJacMax + 1) + 4 * (kJacMax / 2)) +
                           sizeof(int) * 3 * kJacMax);
    SBD_CUDA(ctx, sbd_smem_attr((const void *)jacobi_kernel, ctx->device, (size_t)smem));
    jacobi_kernel<<<1, kJacThreads, smem, ctx->stream>>>(A, k, lda, evals, evecs, max_sweeps, info);
    SBD_LAUNCHED(ctx, "jacobi");
    return SBD_OK;
}

}  // extern "C"
