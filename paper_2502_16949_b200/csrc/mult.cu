// DistMult / ComplEx / RotatE hot path: fused forward on the multiplicative
// incidence layout (gather + times-times row or mulsub row + exact-order score
// + margin hinge + loss) that also emits the per-entry gradient rows, so the
// backward is the same sorted-segment reduce + SGD as the translational path.
//
// Reference (all under /root/reference/proj):
//   build_multiplicative  incidence.hpp:93-121  +1 at head and relation, the
//                         tail +1 (DistMult) or the -1 conjugate marker
//                         (ComplEx, RotATE); head == tail is rejected
//   spmm<TimesTimes>      sparse.hpp:91-106, 244-262: identity, then every
//                         entry in stored (ascending-column) order
//   spmm_mulsub           sparse.hpp:341-365 (RotatE: prod(selecting) - sum(rest))
//   sum_row / sum_real / sum_abs  norms.hpp:76-92 (sequential left-to-right)
//   spmm_product_grad_add sparse.hpp:315-339, spmm_mulsub_grad_add :367-391,
//   modulus_direction     norms.hpp:129-135
//   distmult/complex/rotate_forward, rotate_backward  models.cpp:201-263
//   energy_sign           models.hpp:32-38 (DistMult / ComplEx score
//                         plausibility: the hinge sees -score)
//
// Arithmetic follows the reference bit for bit: complex products in the
// std::complex / Eigen-packet order (re = ar*br - ai*bi, im = ar*bi + ai*br,
// no FMA), the identity (1, 0) multiplied in literally, |q| as glibc's
// hypotf (sqrt of the double-precision sum of squares, rounded once), and
// every score summed sequentially. Complex tables are interleaved (re, im)
// pairs, the reference's std::complex<float> row-major layout.
//
// Gradient rows. For row i with upstream u_i, entry p (head, tail or
// relation column) receives c_p = u_i * others_p (conjugated when p selects,
// ComplEx) or, for RotatE, dq * conj(others_p) / -dq. The forward writes c_p
// into plane p of `res` ([head | tail | relation] x rows x width); the
// segment backward (hrt.cu, kMultRows) sums each column's entries in the
// reference's (pos rows, then neg rows, ascending) order and applies SGD.
// Rows with an inactive hinge contribute u = 0 and are skipped, which changes
// only the sign of exact zeros (as on the translational path).
#include "common.cuh"
#include "kernels.cuh"
#include "multmath.cuh"
#include "primitives.cuh"

namespace skg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr float kEps = 1e-6f;  // kNormEps for 32-bit reals, common.hpp:34

// Gradient rows of one coordinate: head, tail and relation entry.
template <int KIND>
__device__ __forceinline__ void contributions(typename Unit<KIND>::T h, typename Unit<KIND>::T t,
                                              typename Unit<KIND>::T r, bool tail_lo, float u,
                                              typename Unit<KIND>::T& ch, typename Unit<KIND>::T& ct,
                                              typename Unit<KIND>::T& cr) {
  if constexpr (KIND == kDistMult) {
    // others = product of the other two entries in stored order (sparse.hpp:326-332)
    const float lo = tail_lo ? t : h, hi = tail_lo ? h : t;
    const float o_lo = __fmul_rn(hi, r), o_hi = __fmul_rn(lo, r), o_r = __fmul_rn(lo, hi);
    const float c_lo = __fmul_rn(u, o_lo), c_hi = __fmul_rn(u, o_hi);
    ch = tail_lo ? c_hi : c_lo;
    ct = tail_lo ? c_lo : c_hi;
    cr = __fmul_rn(u, o_r);
  } else if constexpr (KIND == kComplEx) {
    const float2 yt = conj2(t);
    const float2 lo = tail_lo ? yt : h, hi = tail_lo ? h : yt;
    const float2 o_lo = cmul(cmul(one2(), hi), r);
    const float2 o_hi = cmul(cmul(one2(), lo), r);
    const float2 o_r = cmul(cmul(one2(), lo), hi);
    const float2 o_h = tail_lo ? o_hi : o_lo, o_t = tail_lo ? o_lo : o_hi;
    ch = scale2(u, conj2(o_h));  // selecting entries take the conjugate (sparse.hpp:333-336)
    ct = scale2(u, o_t);
    cr = scale2(u, conj2(o_r));
  } else {
    // modulus_direction of q, then dq * conj(others) on h and r, -dq on t
    const float2 q = Unit<kRotatE>::q(h, t, r);
    const float m2 = __fadd_rn(__fmul_rn(q.x, q.x), __fmul_rn(q.y, q.y));
    const float inv = __fdiv_rn(u, __fsqrt_rn(__fadd_rn(m2, kEps)));
    const float2 dq = make_float2(__fmul_rn(q.x, inv), __fmul_rn(q.y, inv));
    ch = cmul(dq, conj2(cmul(one2(), r)));
    cr = cmul(dq, conj2(cmul(one2(), h)));
    ct = make_float2(-dq.x, -dq.y);
  }
}

__device__ __forceinline__ bool fin(float a) { return finite_f(a); }
__device__ __forceinline__ bool fin(float2 a) { return finite2(a); }

// 16-byte chunks of a table row: 4 real coordinates or 2 complex ones.
template <int KIND>
struct Chunk {
  static constexpr int NU = KIND == kDistMult ? 4 : 2;  // coordinates per float4
  using T = typename Unit<KIND>::T;
  static __device__ __forceinline__ T get(const float4& v, int k) {
    if constexpr (KIND == kDistMult) {
      return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
    } else {
      return k == 0 ? make_float2(v.x, v.y) : make_float2(v.z, v.w);
    }
  }
  static __device__ __forceinline__ void put(float4& v, int k, T x) {
    if constexpr (KIND == kDistMult) {
      if (k == 0) v.x = x;
      else if (k == 1) v.y = x;
      else if (k == 2) v.z = x;
      else v.w = x;
    } else {
      if (k == 0) v.x = x.x, v.y = x.y;
      else v.z = x.x, v.w = x.y;
    }
  }
};

// A warp owns a tile of 8 (pos, neg) pairs (TRAIN) or 16 rows (SCORE); lanes
// run over the row's coordinates. Per-coordinate score terms are staged in
// shared memory so that lane j then sums row j in the reference's order.
template <int KIND, bool TRAIN, int VEC>
__global__ void __launch_bounds__(kThreads) mult_forward_kernel(const FwdArgs a) {
#ifdef SKG_MULT_NOPAIR
  constexpr bool kPairRounds = false;
#else
  constexpr bool kPairRounds = TRAIN;
#endif
  using U = Unit<KIND>;
  using T = typename U::T;
  extern __shared__ float smem[];
  __shared__ float warp_loss[kWarps];
  if (a.err[0] != 0) return;  // sticky error: nothing runs after the failing batch
  if (a.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) stamp_now(a.stamp_start);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = a.de;                                   // coordinates per row
  const int W = (KIND == kDistMult) ? d : 2 * d;        // floats per table row
  const int S = (d & 1) ? d : d + 1;                    // odd stride: conflict-free row reads
  float* rows = smem + warp * 16 * S;
  constexpr int kUnits = TRAIN ? 8 : 16;
  const int ntiles = (a.B + kUnits - 1) / kUnits;
  const int64_t N = a.N;
  const int nwarps = blockDim.x >> 5;
  float lsum = 0.f;
  uint32_t pend = 0;
  T* P0 = reinterpret_cast<T*>(a.res);

  for (int tile = blockIdx.x * nwarps + warp; tile < ntiles; tile += gridDim.x * nwarps) {
    int h = 0, t = 0, r = 0, row2 = 0;
    bool valid = false;
    if (lane < 16) {
      if (TRAIN) {
        const int p = tile * 8 + (lane & 7);
        const bool neg = lane >= 8;
        valid = p < a.B;
        if (valid) {
          const int4 pq = __ldg(a.pair_ht + p);
          h = neg ? pq.z : pq.x;
          t = neg ? pq.w : pq.y;
          r = __ldg(a.pair_r + p);
          row2 = neg ? a.B + p : p;
        }
      } else {
        const int i = tile * 16 + lane;
        valid = i < a.B;
        if (valid) {
          h = a.H[i];
          t = a.T[i];
          r = a.Rl[i];
          row2 = i;
        }
      }
    }
    const unsigned vmask = __ballot_sync(kFull, valid);

    // ---- per-coordinate score terms of the tile's rows into shared memory
    bool badrow = false;  // lane j: a non-finite term in row j (gradient would be non-finite)
#pragma unroll 1
    for (int j0 = 0; j0 < 16; j0 += 4) {
      // a round's four rows: TRAIN, two (pos, neg) pairs {p, p + 8, p + 1, p + 9}
      // (a pair shares its relation row: loaded once); SCORE, rows j0 .. j0 + 3
      int rowq[4], hj[4], tj[4], rj[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        rowq[q] = kPairRounds ? (j0 >> 1) + (q >> 1) + (q & 1) * 8 : j0 + q;
        hj[q] = __shfl_sync(kFull, h, rowq[q]);
        tj[q] = __shfl_sync(kFull, t, rowq[q]);
        rj[q] = __shfl_sync(kFull, r, rowq[q]);
      }
      bool nf[4] = {false, false, false, false};
      if constexpr (VEC == 4) {
        using CK = Chunk<KIND>;
        const float4* X4 = reinterpret_cast<const float4*>(a.X);
        const int W4 = W >> 2;
        for (int c = lane; c < W4; c += 32) {
          float4 xh[4], xt[4], xr[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!((vmask >> rowq[q]) & 1u)) continue;
            xh[q] = __ldg(X4 + static_cast<size_t>(hj[q]) * W4 + c);
            xt[q] = __ldg(X4 + static_cast<size_t>(tj[q]) * W4 + c);
            if (!kPairRounds || (q & 1) == 0) xr[q] = __ldg(X4 + static_cast<size_t>(N + rj[q]) * W4 + c);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!((vmask >> rowq[q]) & 1u)) continue;
            const float4 xrq = (kPairRounds && (q & 1)) ? xr[q - 1] : xr[q];
#pragma unroll
            for (int k = 0; k < CK::NU; ++k) {
              const T h1 = CK::get(xh[q], k), t1 = CK::get(xt[q], k), r1 = CK::get(xrq, k);
              const float v = U::term(h1, t1, r1, tj[q] < hj[q]);
              nf[q] |= !finite_f(v) || !fin(h1) || !fin(t1) || !fin(r1);
              rows[rowq[q] * S + c * CK::NU + k] = v;
            }
          }
        }
      } else {
        for (int c = lane; c < d; c += 32) {
          T xh[4], xt[4], xr[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!((vmask >> rowq[q]) & 1u)) continue;
            xh[q] = U::load(a.X, hj[q], W, c);
            xt[q] = U::load(a.X, tj[q], W, c);
            xr[q] = U::load(a.X, N + rj[q], W, c);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!((vmask >> rowq[q]) & 1u)) continue;
            const float v = U::term(xh[q], xt[q], xr[q], tj[q] < hj[q]);
            nf[q] |= !finite_f(v) || !fin(xh[q]) || !fin(xt[q]) || !fin(xr[q]);
            rows[rowq[q] * S + c] = v;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool any = __any_sync(kFull, nf[q]);
        if (lane == rowq[q]) badrow = any;
      }
    }
    __syncwarp();

    // ---- exact-order score: lane j sums row j left to right (norms.hpp:76-92)
    float score = 0.f;
    if (lane < 16 && valid) {
      const float* v = rows + lane * S;
      float s = 0.f;
      for (int k = 0; k < d; ++k) s = __fadd_rn(s, v[k]);
      score = s;
    }
    const float energy = a.sign < 0.f ? -score : score;  // energy_sign * score (models.hpp:38)

    float u = 0.f;
    if (TRAIN) {
      // ---- margin hinge on (pos = lane k, neg = lane k + 8), training.cpp:73-94, 117-147
      const float ne = __shfl_down_sync(kFull, energy, 8);
      float term = 0.f;
      bool act = false;
      if (lane < 8 && valid) {
        term = __fsub_rn(__fadd_rn(a.margin, energy), ne);
        act = term > 0.f;  // strict
      }
      const float tk = act ? term : 0.f;
      float tsum = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) tsum = __fadd_rn(tsum, __shfl_sync(kFull, tk, k));
      lsum = __fadd_rn(lsum, tsum);
      act = __shfl_sync(kFull, act, lane & 7) && lane < 16 && valid;
      // upstream = sign * d_pos / sign * d_neg (training.cpp:143-145)
      const float dpn = act ? (lane < 8 ? a.unit : -a.unit) : 0.f;
      u = a.sign < 0.f ? -dpn : dpn;
    } else {
      u = (lane < 16 && valid && a.upstream) ? a.upstream[row2] : 0.f;
    }
    // 0 * a non-finite operand product is NaN in the reference's dense gradient
    if (lane < 16 && valid && badrow && (TRAIN || a.upstream)) pend |= kPendEntity;
    if (lane < 16 && valid) {
      a.scal[row2] = u;
      if (!TRAIN) a.scores[row2] = score;
    }

    // ---- gradient rows of the rows with nonzero upstream (RotatE SCORE: also q)
    const bool want_q = !TRAIN && KIND == kRotatE && a.res_u != nullptr;
    const unsigned wmask = __ballot_sync(kFull, lane < 16 && valid && (u != 0.f || want_q)) & vmask;
    for (unsigned m = wmask; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const int hj = __shfl_sync(kFull, h, j), tj = __shfl_sync(kFull, t, j), rj = __shfl_sync(kFull, r, j);
      const int r2 = __shfl_sync(kFull, row2, j);
      const float uj = __shfl_sync(kFull, u, j);
      bool bad_e = false, bad_r = false;
      if constexpr (VEC == 4) {
        using CK = Chunk<KIND>;
        const float4* X4 = reinterpret_cast<const float4*>(a.X);
        float4* P4 = reinterpret_cast<float4*>(a.res);
        const int W4 = W >> 2;
        for (int c = lane; c < W4; c += 32) {
          const float4 xh = __ldg(X4 + static_cast<size_t>(hj) * W4 + c);
          const float4 xt = __ldg(X4 + static_cast<size_t>(tj) * W4 + c);
          const float4 xr = __ldg(X4 + static_cast<size_t>(N + rj) * W4 + c);
          if constexpr (KIND == kRotatE) {
            if (want_q) {
              float4 qv;
#pragma unroll
              for (int k = 0; k < CK::NU; ++k)
                CK::put(qv, k, Unit<kRotatE>::q(CK::get(xh, k), CK::get(xt, k), CK::get(xr, k)));
              reinterpret_cast<float4*>(a.res_u)[static_cast<size_t>(r2) * W4 + c] = qv;
            }
          }
          if (uj == 0.f) continue;
          float4 vh, vt, vr;
#pragma unroll
          for (int k = 0; k < CK::NU; ++k) {
            T ch, ct, cr;
            contributions<KIND>(CK::get(xh, k), CK::get(xt, k), CK::get(xr, k), tj < hj, uj, ch, ct, cr);
            bad_e |= !fin(ch) || !fin(ct);
            bad_r |= !fin(cr);
            CK::put(vh, k, ch);
            CK::put(vt, k, ct);
            CK::put(vr, k, cr);
          }
          P4[(static_cast<size_t>(0) * a.plane_rows + r2) * W4 + c] = vh;
          P4[(static_cast<size_t>(1) * a.plane_rows + r2) * W4 + c] = vt;
          P4[(static_cast<size_t>(2) * a.plane_rows + r2) * W4 + c] = vr;
        }
      } else {
        for (int c = lane; c < d; c += 32) {
          const T xh = U::load(a.X, hj, W, c), xt = U::load(a.X, tj, W, c), xr = U::load(a.X, N + rj, W, c);
          if constexpr (KIND == kRotatE) {
            if (want_q) reinterpret_cast<float2*>(a.res_u)[static_cast<size_t>(r2) * d + c] = Unit<kRotatE>::q(xh, xt, xr);
          }
          if (uj == 0.f) continue;
          T ch, ct, cr;
          contributions<KIND>(xh, xt, xr, tj < hj, uj, ch, ct, cr);
          bad_e |= !fin(ch) || !fin(ct);
          bad_r |= !fin(cr);
          P0[(static_cast<size_t>(0) * a.plane_rows + r2) * d + c] = ch;
          P0[(static_cast<size_t>(1) * a.plane_rows + r2) * d + c] = ct;
          P0[(static_cast<size_t>(2) * a.plane_rows + r2) * d + c] = cr;
        }
      }
      if (TRAIN || a.upstream) {
        if (__any_sync(kFull, bad_e)) pend |= kPendEntity;
        if (__any_sync(kFull, bad_r)) pend |= kPendRelation;
      }
    }
    __syncwarp();
  }

  // ---- deterministic loss reduction and batch finalization (as hrt_forward)
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&a.err[3], pend);
    __threadfence();
  }
  if (!TRAIN) return;
  if (lane == 0) warp_loss[warp] = lsum;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < nwarps; ++w) b = __fadd_rn(b, warp_loss[w]);
    a.block_partial[blockIdx.x] = b;
    last = ticket_acq_rel(a.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && warp == 0) {
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, a.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, a.loss_div > 0.f ? a.loss_div : static_cast<float>(a.B));
      a.batch_loss[a.batch] = loss;
      if (a.stamp_end) stamp_now(a.stamp_end);
      const uint32_t pflags = *reinterpret_cast<volatile uint32_t*>(&a.err[3]);
      if (!(fabsf(loss) <= 3.402823466e38f)) {
        a.err[1] = a.batch;
        atomicCAS(&a.err[0], 0u, static_cast<uint32_t>(kErrLossNonFinite));
      } else if (pflags) {
        a.err[1] = a.batch;
        atomicCAS(&a.err[0], 0u, static_cast<uint32_t>((pflags & kPendEntity) ? kErrGradEntity : kErrGradRelation));
      }
      a.err[3] = 0;
      *a.counter = 0;
    }
  }
}

constexpr size_t kSmemCap = 200 * 1024;

template <int KIND, bool TRAIN, int VEC>
void launch_t(const FwdArgs& a, int num_sms, cudaStream_t s) {
  const int S = (a.de & 1) ? a.de : a.de + 1;
  const size_t per_warp = static_cast<size_t>(16) * S * sizeof(float);
  if (per_warp > kSmemCap) throw CudaError("mult_forward: embedding dimension too large for the staged tile");
  int wpb = static_cast<int>(kSmemCap / 2 / per_warp);
  wpb = wpb < 1 ? 1 : (wpb > kWarps ? kWarps : wpb);
  const size_t smem = wpb * per_warp;
  const int units = TRAIN ? 8 : 16;
  const int ntiles = (a.B + units - 1) / units;
  int per_sm = static_cast<int>(kSmemCap / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  int grid = (ntiles + wpb - 1) / wpb;
  if (grid > num_sms * per_sm) grid = num_sms * per_sm;
  if (grid < 1) grid = 1;
  mult_forward_kernel<KIND, TRAIN, VEC><<<grid, wpb * 32, smem, s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
}

template <int KIND>
void launch_k(bool train, const FwdArgs& a, int num_sms, cudaStream_t s) {
  // 16-byte chunks when a row is a whole number of them (and the tables are aligned)
  const int W = KIND == kDistMult ? a.de : 2 * a.de;
  const bool v4 = W % 4 == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  if (train) {
    if (v4) launch_t<KIND, true, 4>(a, num_sms, s);
    else launch_t<KIND, true, 1>(a, num_sms, s);
  } else {
    if (v4) launch_t<KIND, false, 4>(a, num_sms, s);
    else launch_t<KIND, false, 1>(a, num_sms, s);
  }
}

template <int KIND, bool TRAIN, int VEC>
void configure_one() {
  SKG_CUDA(cudaFuncSetAttribute(mult_forward_kernel<KIND, TRAIN, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemCap)));
}
template <int KIND>
void configure_k() {
  configure_one<KIND, true, 4>();
  configure_one<KIND, true, 1>();
  configure_one<KIND, false, 4>();
  configure_one<KIND, false, 1>();
}

}  // namespace

void configure_mult_kernels() {
  configure_k<kDistMult>();
  configure_k<kComplEx>();
  configure_k<kRotatE>();
}

void launch_mult_forward(int kind, bool train, const FwdArgs& a, int num_sms, cudaStream_t s) {
  switch (kind) {
    case kDistMult: launch_k<kDistMult>(train, a, num_sms, s); break;
    case kComplEx: launch_k<kComplEx>(train, a, num_sms, s); break;
    case kRotatE: launch_k<kRotatE>(train, a, num_sms, s); break;
    default: throw CudaError("launch_mult_forward: not a multiplicative kind");
  }
}

}  // namespace skg
