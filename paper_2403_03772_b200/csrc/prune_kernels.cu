// prune_kernels.cu — the exact pruned search round (branch and bound over candidates).
//
// causal_order only needs the round's argmin of k_p = sum_q min(0, M_pq)^2 (reference
// ordering.cpp:154-160), not every k. Every term is >= 0, so the sum over any subset of a
// row's pairs is a lower bound of k_p. A round therefore evaluates pairs in stages:
//
//   probe   full rows of the R candidates with the lowest predicted k (k* = the smallest of
//           their exact k) + each other row's T strongest predicted partners
//   refine  rows whose partial k has not passed k* evaluate their top-m predicted partners
//           (m = f u, one stage per fraction f)
//   full    rows still alive evaluate every remaining partner: exact k
//
// and a row is pruned as soon as its partial k exceeds k* (1 + 1e-9): the partial and the
// full sums are FP64 sums of the same non-negative terms, whose orders differ by at most
// u 2^-53 relative, so a pruned row's exact k is strictly larger than k* and it can neither
// win nor tie. The winner is the lowest-position argmin over the rows with exact k, which is
// the argmin of the full round. Every evaluated pair has the bits the exhaustive round gives
// it (same per-pair scales, element math and sample-segment reduction order), so the exact
// k of the surviving rows — the winner's included — are the exhaustive round's bits.
//
// Predictions come from KN (d x d, by variable): the last evaluated min(0, M_pq)^2 of every
// pair, filled completely by the exhaustive round 0 and refreshed with every evaluated pair
// afterwards. Removing one root changes most M_pq only slightly, so last round's strongest
// contributors prune a row after a few pairs (non-roots: usually one pair with an ancestor).
//
// Pair lists are built deterministically (per-row selection in ascending partner order +
// exclusive scan), and evaluated by a cooperative persistent kernel that streams batches of
// 32-pair chunks x sample segments and finalises each batch after a grid barrier, so the
// list length never has to reach the host.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "plg_kernels.h"
#include "plg_math.cuh"
#include "plg_pair.cuh"

namespace cg = cooperative_groups;

namespace plg {

namespace {

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
constexpr double kPruneSlack = 1e-9;  // relative margin over k* (>> u 2^-53)

__device__ __forceinline__ bool is_eval(double m) { return m == m; }  // NaN = not evaluated

__device__ __forceinline__ double kstar_threshold(const PruneArgs& a) {
  return __longlong_as_double(static_cast<long long>(*a.kstar)) * (1.0 + kPruneSlack);
}

// ---- predict: pk[p] = sum_q KN(p, q); collinearity of every pair; state = alive ----
__global__ void __launch_bounds__(256) prune_predict_kernel(const PruneArgs a) {
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= a.u) return;
  const int vp = a.act[p];
  const double* kn = a.KN + static_cast<int64_t>(vp) * a.d;
  double acc = 0.0;
  bool collinear = false;
  for (int q = lane; q < a.u; q += 32) {
    if (q == p) continue;
    const int vq = a.act[q];
    acc += kn[vq];
    if (q > p) {  // the exhaustive round checks every pair (pair_kernel.cu pair_params)
      double s1, bs1, s2, bs2;
      collinear |= !pair_scales(a.C, a.ldc, vp, vq, s1, bs1, s2, bs2);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (__any_sync(0xffffffffu, collinear) && lane == 0) atomicMin(a.err, err_key(a.round, kErrPairCollinear, -1));
  if (lane == 0) {
    a.pk[p] = acc;
    a.state_out[p] = 1;
    a.L[p] = 0.0;
  }
}

// ---- top: the R rows with the lowest pk (ties: lowest position) become full rows ----
constexpr int kTopThreads = 1024;
__global__ void __launch_bounds__(kTopThreads) prune_top_kernel(const PruneArgs a, int R) {
  __shared__ double sv[kTopThreads / 32];
  __shared__ int sp[kTopThreads / 32];
  __shared__ int chosen;
  int* state = a.state_out;
  if (threadIdx.x == 0) *a.kstar = kInfBits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < R && r < a.u; ++r) {
    double best = 0.0;
    int bp = -1;
    for (int p = threadIdx.x; p < a.u; p += kTopThreads) {
      if (state[p] != 1) continue;
      const double v = a.pk[p];
      if (bp < 0 || v < best) {
        best = v;
        bp = p;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (op >= 0 && (bp < 0 || ov < best || (ov == best && op < bp))) {
        best = ov;
        bp = op;
      }
    }
    if (lane == 0) {
      sv[warp] = best;
      sp[warp] = bp;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      int c = -1;
      for (int w = 0; w < kTopThreads / 32; ++w) {
        if (sp[w] >= 0 && (c < 0 || sv[w] < b || (sv[w] == b && sp[w] < c))) {
          b = sv[w];
          c = sp[w];
        }
      }
      chosen = c;
      if (c >= 0) state[c] = 2;
    }
    __syncthreads();
    if (chosen < 0) break;
  }
}

// ---- select: each row's partners for one stage, ascending, into rowsel[p * u + i] ----
constexpr int kSelThreads = 256;
constexpr int kBins = 2049;  // 0: known zero; 1 + biased exponent otherwise (1: unknown marker)

__device__ __forceinline__ int key_bin(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return b == 0 ? 0 : 1 + static_cast<int>(b >> 52);
}

// Block-wide exclusive prefix of a predicate over one 256-wide chunk; returns the chunk total.
__device__ __forceinline__ int block_prefix(bool pred, int* s_warp, int& excl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  if (lane == 0) s_warp[warp] = __popc(bal);
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) {
    const int c = s_warp[w];
    before += (w < warp) ? c : 0;
    total += c;
  }
  excl = before + __popc(bal & ((1u << lane) - 1u));
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kSelThreads) prune_select_kernel(const PruneArgs a, int stage, int m) {
  __shared__ int hist[kBins];
  __shared__ int s_warp[kSelThreads / 32];
  __shared__ int s_cut[2];  // boundary bin, entries of it to take
  const int p = blockIdx.x;
  const int u = a.u;
  const int st = a.state_in[p];
  const double thr = (stage == kStageProbe) ? 0.0 : kstar_threshold(a);
  auto alive_now = [&](int r) { return a.state_in[r] == 1 && a.L[r] <= thr; };
  bool active = false, full = false;
  if (stage == kStageProbe) {
    active = true;
    full = (st == 2);
  } else {
    active = alive_now(p);
    full = (stage == kStageFull);
  }
  if (threadIdx.x == 0) {
    a.state_out[p] = (st == 1 && stage != kStageProbe && !active) ? 0 : st;
    if (!active) a.off[p] = 0;
  }
  if (!active) return;
  const double* md = a.Md + static_cast<int64_t>(p) * u;
  const double* kn = a.KN + static_cast<int64_t>(a.act[p]) * a.d;
  auto eligible = [&](int q) -> bool {
    if (q == p || is_eval(md[q])) return false;
    if (stage == kStageProbe) return full ? !(a.state_in[q] == 2 && q < p) : a.state_in[q] != 2;
    if (stage == kStageFull) return !(q < p && alive_now(q));  // the pair is row q's
    return true;
  };
  int cut_bin = -1, cut_take = 0;  // full: every eligible partner
  if (!full) {
    for (int i = threadIdx.x; i < kBins; i += kSelThreads) hist[i] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < u; q += kSelThreads)
      if (eligible(q)) atomicAdd(&hist[key_bin(kn[a.act[q]])], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // suffix scan from the top bin: the bin where the count reaches m
      const int lane = threadIdx.x;
      constexpr int per = (kBins + 31) / 32;
      const int hi = kBins - 1 - lane * per;  // lane covers bins (hi - per, hi]
      int own = 0;
      for (int b = hi; b > hi - per && b >= 0; --b) own += hist[b];
      int incl = own;  // inclusive prefix over lanes = count in bins >= lane's lowest bin
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int above = incl - own;  // count in bins above this lane's range
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= m);
      if (hit == 0) {
        if (lane == 0) s_cut[0] = -1, s_cut[1] = 0;  // fewer than m eligible: take all
      } else if (lane == __ffs(hit) - 1) {
        int cnt = above, b = hi;
        while (cnt + hist[b] < m) cnt += hist[b--];
        s_cut[0] = b;
        s_cut[1] = m - cnt;
      }
    }
    __syncthreads();
    cut_bin = s_cut[0];
    cut_take = s_cut[1];
  }
  // emit in ascending q: bins above the cut, then the first cut_take of the cut bin
  int* out = a.rowsel + static_cast<int64_t>(p) * u;
  int written = 0, taken_cut = 0;
  for (int base = 0; base < u; base += kSelThreads) {
    const int q = base + threadIdx.x;
    bool sel = false, in_cut = false;
    if (q < u && eligible(q)) {
      if (cut_bin < 0) {
        sel = true;
      } else {
        const int b = key_bin(kn[a.act[q]]);
        sel = b > cut_bin;
        in_cut = (b == cut_bin);
      }
    }
    if (cut_bin >= 0) {
      int rk;
      const int nc = block_prefix(in_cut, s_warp, rk);
      if (in_cut && taken_cut + rk < cut_take) sel = true;
      taken_cut += nc;
    }
    int pos;
    const int ns = block_prefix(sel, s_warp, pos);
    if (sel) out[written + pos] = q;
    written += ns;
  }
  if (threadIdx.x == 0) a.off[p] = written;
}

// ---- scan: off[0..u) counts -> exclusive offsets, off[u] = total ----
__global__ void __launch_bounds__(1024) prune_scan_kernel(const PruneArgs a) {
  __shared__ int s_w[32];
  __shared__ int s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < a.u; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = (i < a.u) ? a.off[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const int excl = s_carry + (warp ? s_w[warp - 1] : 0) + incl - v;
    if (i < a.u) a.off[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.off[a.u] = s_carry;
    atomicAdd(a.evals, static_cast<unsigned long long>(s_carry));
  }
  for (int b = threadIdx.x; b <= s_carry / a.batch; b += blockDim.x) a.work[b] = 0;  // fetch counters
}

// ---- pairs: cooperative persistent evaluation of the list ----
constexpr int kListThreads = 256;

__device__ __forceinline__ void list_entry(const PruneArgs& a, int k, int& p, int& q) {
  int lo = 0, hi = a.u;  // largest p with off[p] <= k (rows with zero entries share offsets)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.off[mid] <= k) lo = mid;
    else hi = mid;
  }
  p = lo;
  q = a.rowsel[static_cast<int64_t>(p) * a.u + (k - a.off[p])];
}

template <bool kClampA>
__device__ __forceinline__ void ede2(double xa, double ya, double s1, double bs1, double s2, double bs2,
                                     EdeAcc& acc1, EdeAcc& acc2, const TabPtr& tp) {
  ede_accumulate<kClampA>(fma(ya, -bs1, xa * s1), acc1, tp);
  ede_accumulate<kClampA>(fma(xa, -bs2, ya * s2), acc2, tp);
}

// Finalise one 32-pair chunk once all its sample segments are in: segments in ascending
// order (finalize_kernel's order), both entropies, then M_pq and M_qp = -M_pq.
__device__ __forceinline__ void finalize_chunk(const PruneArgs& a, const double* part, int base, int m, int chunk,
                                               int lane) {
  const int kk = chunk * 32 + lane;
  if (kk >= m) return;
  int p, q;
  list_entry(a, base + kk, p, q);
  double l1 = 0.0, p1 = 0.0, l2 = 0.0, p2 = 0.0;
  const double2* src = reinterpret_cast<const double2*>(part + static_cast<int64_t>(kk) * 4);
  const int64_t stride = static_cast<int64_t>(a.batch) * 2;  // double2 per segment
  for (int s = 0; s < a.nseg; ++s) {
    const double2 v1 = __ldcg(src);  // written by other SMs: bypass L1
    const double2 v2 = __ldcg(src + 1);
    l1 += v1.x;
    p1 += v1.y;
    l2 += v2.x;
    p2 += v2.y;
    src += stride;
  }
  const double inv_n = 1.0 / static_cast<double>(a.n);
  const double e_pq = entropy_from_sums(l1, p1, inv_n);  // E(p | q)
  const double e_qp = entropy_from_sums(l2, p2, inv_n);  // E(q | p)
  // ordering.cpp:93-94 (kreduce_kernel's expression); M_qp = -M_pq exactly
  const double mpq = (a.H[q] + e_pq) - (a.H[p] + e_qp);
  a.Md[static_cast<int64_t>(p) * a.u + q] = mpq;
  a.Md[static_cast<int64_t>(q) * a.u + p] = -mpq;
}

// Work items (chunk of 32 list entries, sample segment) are fetched dynamically, chunk-major;
// the warp completing a chunk's last segment finalises it, so a batch needs no grid barrier.
// Lists longer than one batch (part-buffer capacity) run batch after batch with a grid
// barrier between them (the kernel is launched cooperatively).
template <bool kClampA>
__global__ void __launch_bounds__(kListThreads, 2) prune_pairs_kernel(const PruneArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  load_tables(smem, a.g_exp, a.g_log);
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const bool skip = (*a.err != kNoError);  // only skips work: every CTA still meets the barriers
  const TabPtr tp = table_ptrs(smem, lane);
  const int total = a.off[a.u];
  const int nbatch = (total + a.batch - 1) / a.batch;
  for (int b = 0; b < nbatch; ++b) {
    if (b > 0) grid.sync();  // every chunk of batch b - 1 is finalised: the part slab is free
    const int base = b * a.batch;
    const int m = min(a.batch, total - base);
    const int chunks = (m + 31) / 32;
    const int items = chunks * a.nseg;
    while (!skip) {
      int it = 0;
      if (lane == 0) it = atomicAdd(&a.work[b], 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= items) break;
      const int chunk = it / a.nseg;
      const int seg = it - chunk * a.nseg;
      const int kk = chunk * 32 + lane;
      if (kk < m) {
        int p, q;
        list_entry(a, base + kk, p, q);
        const int ci = a.act[p], cj = a.act[q];
        double s1, bs1, s2, bs2;
        pair_scales(a.C, a.ldc, ci, cj, s1, bs1, s2, bs2);  // collinear pairs: zeros (flagged by predict)
        const double* wi = a.W + static_cast<int64_t>(ci) * a.ldw;
        const double* wj = a.W + static_cast<int64_t>(cj) * a.ldw;
        const int64_t t0 = static_cast<int64_t>(seg) * a.seg_len;  // multiple of 4: 32-byte aligned
        const int64_t t1 = lmin(a.n, t0 + a.seg_len);
        EdeAcc acc1, acc2;
        int64_t t = t0;
        if (t + 3 < t1) {
          double2 xa = __ldg(reinterpret_cast<const double2*>(wi + t));
          double2 xb = __ldg(reinterpret_cast<const double2*>(wi + t + 2));
          double2 ya = __ldg(reinterpret_cast<const double2*>(wj + t));
          double2 yb = __ldg(reinterpret_cast<const double2*>(wj + t + 2));
#pragma unroll 1
          for (; t + 3 < t1; t += 4) {
            const double2 cxa = xa, cxb = xb, cya = ya, cyb = yb;
            if (t + 7 < t1) {  // prefetch the next 4 samples
              xa = __ldg(reinterpret_cast<const double2*>(wi + t + 4));
              xb = __ldg(reinterpret_cast<const double2*>(wi + t + 6));
              ya = __ldg(reinterpret_cast<const double2*>(wj + t + 4));
              yb = __ldg(reinterpret_cast<const double2*>(wj + t + 6));
            }
            ede2<kClampA>(cxa.x, cya.x, s1, bs1, s2, bs2, acc1, acc2, tp);
            ede2<kClampA>(cxa.y, cya.y, s1, bs1, s2, bs2, acc1, acc2, tp);
            ede2<kClampA>(cxb.x, cyb.x, s1, bs1, s2, bs2, acc1, acc2, tp);
            ede2<kClampA>(cxb.y, cyb.y, s1, bs1, s2, bs2, acc1, acc2, tp);
          }
        }
        for (; t < t1; ++t) ede2<kClampA>(wi[t], wj[t], s1, bs1, s2, bs2, acc1, acc2, tp);
        double2* dst = reinterpret_cast<double2*>(a.part + (static_cast<int64_t>(seg) * a.batch + kk) * 4);
        __stcg(dst, make_double2(acc_lc(acc1), acc_pdf(acc1)));
        __stcg(dst + 1, make_double2(acc_lc(acc2), acc_pdf(acc2)));
      }
      __threadfence();  // release this segment's partials before counting it
      __syncwarp();
      int last = 0;
      if (lane == 0) last = (atomicAdd(&a.done[chunk], 1) == a.nseg - 1);
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();  // acquire the other segments' partials
        finalize_chunk(a, a.part, base, m, chunk, lane);
        if (lane == 0) a.done[chunk] = 0;  // ready for the next batch / launch
      }
    }
  }
}

// ---- bound: partial (or exact) k per row from the evaluated pairs ----
__global__ void __launch_bounds__(256) prune_bound_kernel(const PruneArgs a, int final_pass) {
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= a.u) return;
  if (*a.err != kNoError) return;
  const double* md = a.Md + static_cast<int64_t>(p) * a.u;
  double* kn = final_pass ? a.KN + static_cast<int64_t>(a.act[p]) * a.d : nullptr;
  // kreduce_kernel's lane-strided order: for a fully evaluated row this is its exact k bits
  double acc = 0.0;
  for (int q = lane; q < a.u; q += 32) {
    if (q == p) continue;
    const double mi = md[q];
    if (!is_eval(mi)) continue;
    const double c = (mi < 0.0) ? mi : 0.0;
    acc = __dadd_rn(acc, __dmul_rn(c, c));
    if (kn) kn[a.act[q]] = __dmul_rn(c, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
  const int st = a.state_in[p];
  if (final_pass) {
    a.k[p] = (st >= 1) ? acc : __longlong_as_double(static_cast<long long>(kInfBits));
  } else {
    a.L[p] = acc;
    if (st == 2) atomicMin(a.kstar, static_cast<unsigned long long>(__double_as_longlong(acc)));
  }
}

template <bool kClampA>
int pairs_grid_for() {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(prune_pairs_kernel<kClampA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableBytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, prune_pairs_kernel<kClampA>, kListThreads, kTableBytes);
    grid = sms * (per > 0 ? per : 1);
  }
  return grid;
}

template <bool kClampA>
void launch_pairs_cfg(const PruneArgs& a, cudaStream_t s) {
  const int grid = pairs_grid_for<kClampA>();
  PruneArgs args = a;
  void* params[] = {&args};
  cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(prune_pairs_kernel<kClampA>), dim3(grid),
                              dim3(kListThreads), params, kTableBytes, s);
}

}  // namespace

void launch_prune_predict(const PruneArgs& a, cudaStream_t s) {
  prune_predict_kernel<<<(a.u + 7) / 8, 256, 0, s>>>(a);
}

void launch_prune_top(const PruneArgs& a, int R, cudaStream_t s) {
  prune_top_kernel<<<1, kTopThreads, 0, s>>>(a, R);
}

void launch_prune_select(const PruneArgs& a, int stage, int m, cudaStream_t s) {
  prune_select_kernel<<<a.u, kSelThreads, 0, s>>>(a, stage, m);
}

void launch_prune_scan(const PruneArgs& a, cudaStream_t s) { prune_scan_kernel<<<1, 1024, 0, s>>>(a); }

void launch_prune_pairs(const PruneArgs& a, cudaStream_t s) {
  if (a.n > 90000) launch_pairs_cfg<true>(a, s);
  else launch_pairs_cfg<false>(a, s);
}

void launch_prune_bound(const PruneArgs& a, bool final_pass, cudaStream_t s) {
  prune_bound_kernel<<<(a.u + 7) / 8, 256, 0, s>>>(a, final_pass ? 1 : 0);
}

int prune_pairs_grid() { return pairs_grid_for<false>(); }

}  // namespace plg
