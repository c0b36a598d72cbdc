// cs_fit.cu — batched least-squares GBDT fit on the device:
// fit_gbdt (gbdt.cpp:123-171) with TreeBuilder::build (gbdt.cpp:50-118) for
// many independent training sets at once, one CTA per model, with results
// identical to the reference's (the model JSON is byte-identical).
//
// Per model the CTA keeps in shared memory (global scratch when a training
// set is too large): residuals, the current row partition (ascending row ids
// per node, as the reference's stable index split keeps them), per-feature
// gathered keys and sort permutations, and the cached root permutation.
// Trees grow level by level (nodes of one level are independent), and node
// ids / importance are then assigned in the reference's pre-order.
//
// Bit-exactness:
//  * every sum the reference computes sequentially stays sequential, in the
//    same order (node totals in row order; prefix sums in sorted order; the
//    base mean; importance in pre-order, tree after tree);
//  * the sorted order is libstdc++'s std::sort restated (cs_introsort.h), so
//    equal feature values keep the reference's tie order;
//  * the root's sort input is the same every tree (keys only depend on the
//    row order), so its permutation is computed once per model;
//  * the split choice runs features in order with the running best, the
//    1e-12 margins and strict comparisons of gbdt.cpp:83-88;
//  * compiled with --fmad=false (no contractions), IEEE division.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "cs_fit.h"
#include "cs_introsort.h"

namespace {

constexpr int kFitThreads = 512;
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kMaxDepth = 8;  // node table: 2^(kMaxDepth+1) - 1 entries

struct BNode {
  uint32_t start, len;  // segment of the row partition
  uint32_t n_left;      // rows going left (internal nodes)
  int32_t feature;      // -1: leaf
  int32_t left, right;  // BFS ids of the children
  double sum;           // row-order total of the residuals
  double thr, gain;
};

// the sorted element: (feature value, row) — the reference sorts (feature
// value, residual) pairs with a comparator on the value only
struct KP {
  double key;
  uint32_t row, pad;
};
struct KPLess {
  __device__ __forceinline__ bool operator()(const KP& a, const KP& b) const { return a.key < b.key; }
};

struct FitArgs {
  uint32_t n_models, F;
  const uint64_t* off;
  const double* x;      // column-major per model
  const double* y;
  KP* root;             // per row and feature: the root's sorted (value, row) pairs
  uint8_t* scratch;     // global working memory for models beyond the smem budget
  const uint64_t* scratch_off;  // per model; UINT64_MAX = shared memory
  uint32_t n_trees, max_depth, min_leaf, node_stride;
  double lr;
  cs_tree_node* nodes;
  uint32_t* n_nodes;
  double* base;
  uint8_t* degenerate;
  double* importance;
  unsigned long long* prof;  // optional per-phase cycle totals (block 0), CS_FIT_PROFILE
};

__host__ __device__ inline uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t{15}; }
__host__ __device__ inline uint64_t work_cap(uint64_t n, uint64_t F) { return F * n / 16 + 64; }
__host__ __device__ inline uint64_t final_cap(uint64_t n, uint64_t F) { return F * n / 2 + 64; }

// working-memory layout of one model with n rows, F features
struct Layout {
  uint64_t r, pred, kp, g, idx_a, idx_b, nodes, work_a, work_b, fin, total;
  __host__ __device__ Layout(uint64_t n, uint64_t F, uint64_t max_nodes) {
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) {
      const uint64_t at = o;
      o = align16(o + bytes);
      return at;
    };
    r = take(8 * n);
    pred = take(8 * n);
    kp = take(sizeof(KP) * F * n);
    g = take(8 * F * n);
    idx_a = take(4 * n);
    idx_b = take(4 * n);
    nodes = take(sizeof(BNode) * max_nodes);
    work_a = take(sizeof(cs_sort::Range) * work_cap(n, F));
    work_b = take(sizeof(cs_sort::Range) * work_cap(n, F));
    fin = take(sizeof(cs_sort::Range) * final_cap(n, F));
    total = o;
  }
};

// libstdc++'s __unguarded_partition_pivot (cs_introsort.h) on kp[first, last)
// by one warp.  The sequential scans swap the i-th left stopper (ascending,
// key >= pivot) with the i-th right stopper (descending, key <= pivot) while
// l_i < r_i; for those i every position a scan passes is still unmodified
// (earlier swaps touched only l_j < l_i and r_j > r_i), so the stoppers are
// those of the input.  The warp lists both stopper sequences of the input
// with ballots, finds K = the first i with l_i >= r_i, performs the K swaps
// in parallel and returns min(l_{K+1}, r_K), where the sequential scan stops.
// `scratch` holds 2 * (last - first) u32 (the range's slice of the gain array).
__device__ uint32_t warp_partition(KP* kp, uint32_t first, uint32_t last, uint32_t* scratch, int lane) {
  const KPLess lt;
  if (lane == 0) cs_sort::move_median_to_first(kp, first, first + 1, first + (last - first) / 2, last - 1, lt);
  __syncwarp();
  const double pv = kp[first].key;
  const uint32_t m = last - first;
  uint32_t* Ls = scratch;
  uint32_t* Rs = scratch + m;
  const uint32_t below = (1u << lane) - 1u;
  uint32_t nL = 0, nR = 0;
  for (uint32_t b = first + 1; b < last; b += 32) {
    const uint32_t p = b + lane;
    const bool f = p < last && !(kp[p].key < pv);
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (f) Ls[nL + __popc(bal & below)] = p;
    nL += __popc(bal);
  }
  for (uint32_t e = last; e > first + 1; e = e > first + 33 ? e - 32 : first + 1) {
    const bool valid = e - 1 >= first + 1 + (uint32_t)lane && (uint32_t)lane < e - 1 - first;
    const uint32_t p = valid ? e - 1 - lane : first;
    const bool f = valid && !(pv < kp[p].key);
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (f) Rs[nR + __popc(bal & below)] = p;
    nR += __popc(bal);
  }
  __syncwarp();
  const uint32_t np = nL < nR ? nL : nR;
  uint32_t K = 0;
  for (uint32_t i0 = 0; i0 < np; i0 += 32) {  // l_i < r_i holds for a prefix of i
    const uint32_t i = i0 + lane;
    const uint32_t bal = __ballot_sync(0xffffffffu, i < np && Ls[i] < Rs[i]);
    K += __popc(bal);
    if (bal != 0xffffffffu) break;
  }
  for (uint32_t i = lane; i < K; i += 32) {
    const KP t = kp[Ls[i]];
    kp[Ls[i]] = kp[Rs[i]];
    kp[Rs[i]] = t;
  }
  uint32_t cut = K < nL ? Ls[K] : last;
  if (K > 0 && Rs[K - 1] < cut) cut = Rs[K - 1];
  __syncwarp();
  return cut;
}

// s = ((s + v[0]) + v[1]) + ... in order; loads are issued 8 ahead
__device__ __forceinline__ double seq_sum(const double* v, uint32_t len) {
  double s = 0.0;
  uint32_t k = 0;
  for (; k + 8 <= len; k += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = v[k + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += t[u];
  }
  for (; k < len; ++k) s += v[k];
  return s;
}
// v[k] = v[0] + ... + v[k] (sequential left-to-right sums), in place
__device__ __forceinline__ void seq_prefix(double* v, uint32_t len) {
  double s = 0.0;
  uint32_t k = 0;
  for (; k + 8 <= len; k += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = v[k + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s += t[u];
      v[k + u] = s;
    }
  }
  for (; k < len; ++k) {
    s += v[k];
    v[k] = s;
  }
}

__global__ void __launch_bounds__(kFitThreads, 1) k_gbdt_fit(FitArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  long long t_mark = clock64();
  auto mark = [&](int phase) {
    if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) {
      const long long now = clock64();
      a.prof[phase] += (unsigned long long)(now - t_mark);
      t_mark = now;
    }
  };
  __shared__ double s_mean, s_lo, s_hi;
  __shared__ uint32_t s_nn, s_lvl, s_nwork[2], s_nfin;
  const uint32_t m = blockIdx.x;
  const uint64_t o = a.off[m];
  const uint32_t n = (uint32_t)(a.off[m + 1] - o);
  const uint32_t F = a.F, D = a.max_depth, min_leaf = a.min_leaf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // sequential tasks (one per thread) are dealt to lane 0 of every warp
  // first, then lane 1, ...: tasks on lanes of one warp diverge and run one
  // after another, tasks on different warps run side by side
  const uint32_t task = (uint32_t)lane * kFitWarps + (uint32_t)warp;
  const double* xm = a.x + o * F;  // feature f: xm + f * n
  const double* ym = a.y + o;
  KP* root = a.root + o * F;
  const uint32_t max_nodes = (2u << D) - 1u;
  const Layout L(n, F, max_nodes);
  uint8_t* w = a.scratch_off[m] == ~0ull ? smem : a.scratch + a.scratch_off[m];
  double* r = (double*)(w + L.r);
  double* pred = (double*)(w + L.pred);
  KP* kp = (KP*)(w + L.kp);
  double* g = (double*)(w + L.g);
  uint32_t* idx = (uint32_t*)(w + L.idx_a);
  uint32_t* idx_next = (uint32_t*)(w + L.idx_b);
  BNode* nd = (BNode*)(w + L.nodes);
  cs_sort::Range* work[2] = {(cs_sort::Range*)(w + L.work_a), (cs_sort::Range*)(w + L.work_b)};
  cs_sort::Range* fin = (cs_sort::Range*)(w + L.fin);
  cs_tree_node* out_nodes = a.nodes + (uint64_t)m * a.n_trees * a.node_stride;
  uint32_t* out_count = a.n_nodes + (uint64_t)m * a.n_trees;
  double* imp = a.importance + (uint64_t)m * F;
  const KPLess lt;

  if (tid == 0) {  // base = mean(y), degenerate when every target is equal (gbdt.cpp:132-143)
    double s = 0.0, lo = n ? ym[0] : 0.0, hi = lo;
    for (uint32_t i = 0; i < n; ++i) {
      s += ym[i];
      lo = ym[i] < lo ? ym[i] : lo;
      hi = ym[i] > hi ? ym[i] : hi;
    }
    s_mean = s / (double)n;
    s_lo = lo;
    s_hi = hi;
    for (uint32_t f = 0; f < F; ++f) imp[f] = 0.0;
  }
  __syncthreads();
  if (n == 0) return;
  if (s_lo == s_hi) {
    if (tid == 0) {
      a.base[m] = s_lo;
      a.degenerate[m] = 1;
    }
    for (uint32_t t = tid; t < a.n_trees; t += kFitThreads) out_count[t] = 0;
    return;
  }
  if (tid == 0) {
    a.base[m] = s_mean;
    a.degenerate[m] = 0;
  }
  const double mean = s_mean;
  for (uint32_t i = tid; i < n; i += kFitThreads) pred[i] = mean;
  // the root's sorted pairs: same input (rows in order) for every tree
  for (uint32_t q = tid; q < F * n; q += kFitThreads) root[q] = KP{xm[q], q % n, 0u};
  __syncthreads();
  for (uint32_t f = task; f < F; f += kFitThreads) cs_sort::sort_with(root + (uint64_t)f * n, n, lt);
  __syncthreads();

  for (uint32_t t = 0; t < a.n_trees; ++t) {
    for (uint32_t i = tid; i < n; i += kFitThreads) {
      r[i] = ym[i] - pred[i];
      idx[i] = i;
    }
    if (tid == 0) {
      nd[0] = BNode{0, n, 0, -1, -1, -1, 0.0, 0.0, 0.0};
      s_nn = 1;
      s_lvl = 0;
    }
    __syncthreads();
    mark(0);
    for (uint32_t d = 0;; ++d) {
      const uint32_t lb = s_lvl, le = s_nn;
      if (lb == le) break;
      auto splittable = [&](uint32_t j) { return d < D && (uint64_t)nd[j].len >= 2ull * min_leaf; };
      // (A) node totals in row order (gbdt.cpp:51-53): residuals gathered
      // into row order first, then one sequential sum per node
      for (uint32_t j = lb; j < le; ++j) {
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        for (uint32_t k = tid; k < len; k += kFitThreads) g[s0 + k] = r[idx[s0 + k]];
      }
      if (tid == 0) {
        s_nwork[0] = 0;
        s_nfin = 0;
      }
      __syncthreads();
      for (uint32_t j = lb + task; j < le; j += kFitThreads) {
        nd[j].sum = seq_sum(g + nd[j].start, nd[j].len);
        nd[j].feature = -1;
      }
      __syncthreads();
      mark(1);
      // (B) per feature: (value, row) pairs in row order, the sort's input;
      // the root's are sorted once per model
      for (uint32_t j = lb; j < le; ++j) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        for (uint32_t q = tid; q < F * len; q += kFitThreads) {
          const uint32_t f = q / len, k = q - f * len;
          if (d == 0) {
            kp[(uint64_t)f * n + k] = root[(uint64_t)f * n + k];
          } else {
            const uint32_t row = idx[s0 + k];
            kp[(uint64_t)f * n + s0 + k] = KP{xm[(uint64_t)f * n + row], row, 0u};
          }
        }
        if (d > 0 && tid < (int)F) {
          const uint32_t b0 = (uint32_t)tid * n + s0;
          if (len > (uint32_t)cs_sort::kThreshold) work[0][atomicAdd(&s_nwork[0], 1u)] = cs_sort::start(b0, len);
          else if (len > 1) fin[atomicAdd(&s_nfin, 1u)] = cs_sort::Range{b0, b0 + len, 0u};
        }
      }
      __syncthreads();
      mark(2);
      if (d > 0) {
        // (S) std::sort of every (node, feature) segment as independent range
        // steps (cs_introsort.h): the partition tree level by level, then
        // every final range's insertion sort
        int cur = 0;
        while (true) {
          const uint32_t nw = s_nwork[cur];
          if (nw == 0) break;
          if (tid == 0) s_nwork[cur ^ 1] = 0;
          __syncthreads();
          for (uint32_t q = warp; q < nw; q += kFitWarps) {  // a warp per range
            const cs_sort::Range rg = work[cur][q];
            if (rg.depth == 0) {  // depth limit: heap sort (sorted, nothing left)
              if (lane == 0) cs_sort::heap_sort(kp + rg.first, rg.last - rg.first, lt);
              continue;
            }
            const uint32_t cut = warp_partition(kp, rg.first, rg.last, (uint32_t*)(g + rg.first), lane);
            if (lane == 0) {
              const cs_sort::Range out[2] = {{rg.first, cut, rg.depth - 1}, {cut, rg.last, rg.depth - 1}};
              for (int i = 0; i < 2; ++i) {
                const uint32_t len = out[i].last - out[i].first;
                if (len > (uint32_t)cs_sort::kThreshold) work[cur ^ 1][atomicAdd(&s_nwork[cur ^ 1], 1u)] = out[i];
                else if (len > 1) fin[atomicAdd(&s_nfin, 1u)] = out[i];
              }
            }
          }
          __syncthreads();
          cur ^= 1;
        }
        mark(3);
        const uint32_t nf = s_nfin;
        for (uint32_t q = task; q < nf; q += kFitThreads)
          cs_sort::insertion_sort(kp, fin[q].first, fin[q].last, lt);
        __syncthreads();
        mark(4);
      }
      // (C1) left prefix sums in sorted order (gbdt.cpp:65-67): residuals
      // gathered into sorted order, then one sequential sum per (node, feature)
      for (uint32_t j = lb; j < le; ++j) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        for (uint32_t q = tid; q < F * len; q += kFitThreads) {
          const uint32_t f = q / len, k = q - f * len;
          g[(uint64_t)f * n + s0 + k] = r[kp[(uint64_t)f * n + s0 + k].row];
        }
      }
      __syncthreads();
      for (uint32_t q = task; q < (le - lb) * F; q += kFitThreads) {
        const uint32_t j = lb + q / F, f = q % F;
        if (!splittable(j)) continue;
        seq_prefix(g + (uint64_t)f * n + nd[j].start, nd[j].len - 1);
      }
      __syncthreads();
      mark(5);
      // (C2) candidate gains, all in parallel (gbdt.cpp:68-80); -1 marks a non-candidate
      for (uint32_t j = lb; j < le; ++j) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        const double sum = nd[j].sum, cnt = (double)len;
        for (uint32_t q = tid; q < F * (len - 1); q += kFitThreads) {
          const uint32_t f = q / (len - 1), k = q - f * (len - 1);
          const KP* P = kp + (uint64_t)f * n + s0;
          double* G = g + (uint64_t)f * n + s0;
          const uint32_t ln = k + 1, rn = len - ln;
          double gv = -1.0;
          if (P[k].key != P[k + 1].key && ln >= min_leaf && rn >= min_leaf) {
            const double lsum = G[k], rsum = sum - lsum;
            gv = lsum * lsum / (double)ln + rsum * rsum / (double)rn - sum * sum / cnt;
          }
          G[k] = gv;
        }
      }
      __syncthreads();
      mark(6);
      // (C3) the reference's running best over features then positions
      // (gbdt.cpp:83-88): best is replaced when g > best + 1e-12.  Every
      // earlier candidate c satisfied c <= best + 1e-12 at its turn, so best
      // >= (max of earlier candidates) - 1e-12 and an accepted candidate is a
      // strict prefix maximum.  A warp per node scans the candidates with a
      // running max and replays the chain on the strict prefix maxima only,
      // in order, which gives the sequential result.
      for (uint32_t j = lb + warp; j < le; j += kFitWarps) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len, per = len - 1, total = F * per;
        double best_gain = 0.0, run_max = -1.0;
        uint32_t best_q = 0;
        bool found = false;
        for (uint32_t q0 = 0; q0 < total; q0 += 32) {
          const uint32_t q = q0 + lane;
          double gv = -1.0;
          if (q < total) {
            const uint32_t f = q / per, k = q - f * per;
            gv = g[(uint64_t)f * n + s0 + k];
          }
          double incl = gv;  // inclusive max scan over the chunk
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = fmax(incl, y);
          }
          double excl = __shfl_up_sync(0xffffffffu, incl, 1);
          if (lane == 0) excl = -1.0;
          excl = fmax(excl, run_max);
          uint32_t cand = __ballot_sync(0xffffffffu, q < total && gv > excl);
          // every strict prefix maximum clears the previous one by more than
          // the margin: each is accepted, the last one ends the chunk
          // (best <= max(earlier candidates, 0): the chain starts at 0)
          const uint32_t wide = __ballot_sync(0xffffffffu, q < total && gv > fmax(excl, 0.0) + 1e-12);
          if (cand && wide == cand) {
            const int l = 31 - __clz(cand);
            best_gain = __shfl_sync(0xffffffffu, gv, l);
            best_q = q0 + l;
            found = true;
            cand = 0;
          }
          while (cand) {  // replay the chain on the strict prefix maxima, in order
            const int l = __ffs(cand) - 1;
            cand &= cand - 1;
            const double c = __shfl_sync(0xffffffffu, gv, l);
            if (c > best_gain + 1e-12) {
              best_gain = c;
              best_q = q0 + l;
              found = true;
            }
          }
          run_max = fmax(run_max, __shfl_sync(0xffffffffu, incl, 31));
        }
        if (lane == 0 && found && best_gain > 1e-12) {
          const uint32_t bf = best_q / per, bk = best_q - bf * per;
          const KP* P = kp + (uint64_t)bf * n + s0;
          nd[j].feature = (int32_t)bf;
          nd[j].thr = 0.5 * (P[bk].key + P[bk + 1].key);
          nd[j].gain = best_gain;
        }
      }
      __syncthreads();
      mark(7);
      // (D) stable split of each internal node's rows (gbdt.cpp:97-104), warp per node
      for (uint32_t j = lb + warp; j < le; j += kFitWarps) {
        if (nd[j].feature < 0) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        const double* X = xm + (uint64_t)nd[j].feature * n;
        const double thr = nd[j].thr;
        uint32_t nl = 0;
        for (uint32_t k0 = 0; k0 < len; k0 += 32) {
          const uint32_t k = k0 + lane;
          const uint32_t i = k < len ? idx[s0 + k] : 0u;
          const bool go_left = k < len && X[i] <= thr;
          const uint32_t bl = __ballot_sync(0xffffffffu, go_left);
          if (go_left) idx_next[s0 + nl + __popc(bl & ((1u << lane) - 1u))] = i;
          nl += __popc(bl);
        }
        uint32_t nr = 0;
        for (uint32_t k0 = 0; k0 < len; k0 += 32) {
          const uint32_t k = k0 + lane;
          const uint32_t i = k < len ? idx[s0 + k] : 0u;
          const bool go_right = k < len && !(X[i] <= thr);
          const uint32_t br = __ballot_sync(0xffffffffu, go_right);
          if (go_right) idx_next[s0 + nl + nr + __popc(br & ((1u << lane) - 1u))] = i;
          nr += __popc(br);
        }
        if (lane == 0) nd[j].n_left = nl;
      }
      __syncthreads();
      mark(8);
      if (tid == 0) {  // children in BFS order
        uint32_t nn = le;
        for (uint32_t j = lb; j < le; ++j) {
          if (nd[j].feature < 0) continue;
          const uint32_t s0 = nd[j].start, nl = nd[j].n_left;
          nd[j].left = (int32_t)nn;
          nd[nn++] = BNode{s0, nl, 0, -1, -1, -1, 0.0, 0.0, 0.0};
          nd[j].right = (int32_t)nn;
          nd[nn++] = BNode{s0 + nl, nd[j].len - nl, 0, -1, -1, -1, 0.0, 0.0, 0.0};
        }
        s_lvl = le;
        s_nn = nn;
      }
      // rows of the next level live in idx_next (only split segments matter)
      uint32_t* tmp = idx;
      idx = idx_next;
      idx_next = tmp;
      __syncthreads();
      mark(9);
    }
    // pre-order ids and importance (the reference's recursion order)
    if (tid == 0) {
      int32_t stack[2 * kMaxDepth + 4];
      int32_t pre[1 << (kMaxDepth + 1)];
      int sp = 0, next = 0;
      stack[sp++] = 0;
      while (sp) {  // assign ids
        const int32_t j = stack[--sp];
        pre[j] = next++;
        if (nd[j].feature >= 0) {
          imp[nd[j].feature] += nd[j].gain;
          stack[sp++] = nd[j].right;
          stack[sp++] = nd[j].left;
        }
      }
      cs_tree_node* outt = out_nodes + (uint64_t)t * a.node_stride;
      for (uint32_t j = 0; j < s_nn; ++j) {
        cs_tree_node c;
        c.reserved = 0;
        if (nd[j].feature >= 0) {
          c.feature = nd[j].feature;
          c.left = pre[nd[j].left];
          c.right = pre[nd[j].right];
          c.threshold = nd[j].thr;
          c.value = 0.0;
        } else {
          c.feature = -1;
          c.left = -1;
          c.right = -1;
          c.threshold = 0.0;
          c.value = nd[j].sum / (double)nd[j].len;  // node_mean (gbdt.cpp:52-53)
        }
        outt[pre[j]] = c;
      }
      out_count[t] = s_nn;
    }
    // prediction update (gbdt.cpp:155-156)
    for (uint32_t i = tid; i < n; i += kFitThreads) {
      int32_t j = 0;
      while (nd[j].feature >= 0) j = xm[(uint64_t)nd[j].feature * n + i] <= nd[j].thr ? nd[j].left : nd[j].right;
      pred[i] = pred[i] + a.lr * (nd[j].sum / (double)nd[j].len);
    }
    __syncthreads();
    mark(10);
  }
}

struct DevMem {
  void* p = nullptr;
  ~DevMem() {
    if (p) cudaFree(p);
  }
};

}  // namespace

int gbdt_fit_device(int device, GbdtBatch& b, std::string& err) {
  const uint32_t M = static_cast<uint32_t>(b.off.size() ? b.off.size() - 1 : 0);
  const uint32_t F = b.n_features;
  if (M == 0) return CS_OK;
  if (b.params.max_depth > static_cast<uint64_t>(kMaxDepth)) {
    err = "device fit supports max_depth <= " + std::to_string(kMaxDepth);
    return CS_E_UNSUPPORTED;
  }
  if (F == 0 || F > 8 || b.params.n_trees > (1u << 20)) {
    err = "device fit: 1..8 features, at most 2^20 trees";
    return CS_E_UNSUPPORTED;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    err = "cudaSetDevice";
    return CS_E_CUDA;
  }
  const uint32_t D = static_cast<uint32_t>(b.params.max_depth);
  const uint32_t max_nodes = (2u << D) - 1u;
  b.node_stride = max_nodes;
  // shared-memory budget: models that fit run from shared memory
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const uint64_t smem_budget = static_cast<uint64_t>(std::max(0, smem_optin - 1024));
  uint64_t smem_need = 0, scratch_total = 0;
  std::vector<uint64_t> scratch_off(M, ~0ull);
  for (uint32_t m = 0; m < M; ++m) {
    const uint64_t n = b.off[m + 1] - b.off[m];
    if (n > 0xffffffffull) {
      err = "device fit: too many rows";
      return CS_E_UNSUPPORTED;
    }
    const Layout L(n, F, max_nodes);
    if (L.total <= smem_budget) {
      smem_need = std::max(smem_need, L.total);
    } else {
      scratch_off[m] = scratch_total;
      scratch_total += align16(L.total);
    }
  }
  const uint64_t rows = b.off[M];
  DevMem d_off, d_x, d_y, d_root, d_scr, d_scr_off, d_nodes, d_cnt, d_base, d_deg, d_imp;
  auto alloc = [&](DevMem& x, size_t bytes) { return cudaMalloc(&x.p, std::max<size_t>(bytes, 16)) == cudaSuccess; };
  const size_t node_count = static_cast<size_t>(M) * b.params.n_trees * max_nodes;
  if (!alloc(d_off, (M + 1) * 8) || !alloc(d_x, rows * F * 8) || !alloc(d_y, rows * 8) ||
      !alloc(d_root, rows * F * sizeof(KP)) || !alloc(d_scr, scratch_total) || !alloc(d_scr_off, M * 8) ||
      !alloc(d_nodes, node_count * sizeof(cs_tree_node)) ||
      !alloc(d_cnt, static_cast<size_t>(M) * b.params.n_trees * 4) || !alloc(d_base, M * 8) ||
      !alloc(d_deg, M) || !alloc(d_imp, static_cast<size_t>(M) * F * 8)) {
    err = "cudaMalloc(fit)";
    return CS_E_CUDA;
  }
  cudaMemcpy(d_off.p, b.off.data(), (M + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x.p, b.x_col.data(), rows * F * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_y.p, b.y.data(), rows * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_scr_off.p, scratch_off.data(), M * 8, cudaMemcpyHostToDevice);
  FitArgs a{};
  a.n_models = M;
  a.F = F;
  a.off = static_cast<const uint64_t*>(d_off.p);
  a.x = static_cast<const double*>(d_x.p);
  a.y = static_cast<const double*>(d_y.p);
  a.root = static_cast<KP*>(d_root.p);
  a.scratch = static_cast<uint8_t*>(d_scr.p);
  a.scratch_off = static_cast<const uint64_t*>(d_scr_off.p);
  a.n_trees = static_cast<uint32_t>(b.params.n_trees);
  a.max_depth = D;
  a.min_leaf = static_cast<uint32_t>(std::min<uint64_t>(b.params.min_samples_leaf, 0xffffffffull));
  a.node_stride = max_nodes;
  a.lr = b.params.learning_rate;
  a.nodes = static_cast<cs_tree_node*>(d_nodes.p);
  a.n_nodes = static_cast<uint32_t*>(d_cnt.p);
  a.base = static_cast<double*>(d_base.p);
  a.degenerate = static_cast<uint8_t*>(d_deg.p);
  a.importance = static_cast<double*>(d_imp.p);
  DevMem d_prof;
  const bool prof = std::getenv("CS_FIT_PROFILE") != nullptr;
  if (prof && alloc(d_prof, 16 * 8)) {
    cudaMemset(d_prof.p, 0, 16 * 8);
    a.prof = static_cast<unsigned long long*>(d_prof.p);
  }
  cudaFuncSetAttribute(k_gbdt_fit, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_need));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_gbdt_fit<<<M, kFitThreads, smem_need>>>(a);
  cudaEventRecord(e1);
  const cudaError_t ce = cudaEventSynchronize(e1);
  cudaEventElapsedTime(&b.device_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ce != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    err = std::string("k_gbdt_fit: ") + cudaGetErrorString(ce);
    return CS_E_CUDA;
  }
  if (a.prof) {
    unsigned long long h[16];
    cudaMemcpy(h, a.prof, sizeof h, cudaMemcpyDeviceToHost);
    static const char* kPhase[] = {"residuals", "sums", "gather", "sort", "insertion", "prefix",
                                   "gains", "select", "partition", "children", "tree_out+predict"};
    for (int i = 0; i < 11; ++i) std::fprintf(stderr, "fit phase %-16s %12llu cycles\n", kPhase[i], h[i]);
  }
  b.base.resize(M);
  b.degenerate.resize(M);
  b.importance.resize(static_cast<size_t>(M) * F);
  b.nodes.resize(node_count);
  b.n_nodes.resize(static_cast<size_t>(M) * b.params.n_trees);
  cudaMemcpy(b.base.data(), d_base.p, M * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.degenerate.data(), d_deg.p, M, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.importance.data(), d_imp.p, static_cast<size_t>(M) * F * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.nodes.data(), d_nodes.p, node_count * sizeof(cs_tree_node), cudaMemcpyDeviceToHost);
  cudaMemcpy(b.n_nodes.data(), d_cnt.p, b.n_nodes.size() * 4, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess) {
    err = "fit read-back";
    return CS_E_CUDA;
  }
  return CS_OK;
}
