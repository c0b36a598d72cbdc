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
#include <string>

#include "cs_fit.h"
#include "cs_introsort.h"

namespace {

constexpr int kFitThreads = 256;
constexpr int kMaxDepth = 8;  // node table: 2^(kMaxDepth+1) - 1 entries

struct BNode {
  uint32_t start, len;  // segment of the row partition
  uint32_t n_left;      // rows going left (internal nodes)
  int32_t feature;      // -1: leaf
  int32_t left, right;  // BFS ids of the children
  double sum;           // row-order total of the residuals
  double thr, gain;
};

struct FitArgs {
  uint32_t n_models, F;
  const uint64_t* off;
  const double* x;      // column-major per model
  const double* y;
  double* pred;         // per row
  uint8_t* scratch;     // global working memory for models beyond the smem budget
  const uint64_t* scratch_off;  // per model; UINT64_MAX = shared memory
  uint32_t n_trees, max_depth, min_leaf, node_stride;
  double lr;
  cs_tree_node* nodes;
  uint32_t* n_nodes;
  double* base;
  uint8_t* degenerate;
  double* importance;
};

__host__ __device__ inline uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t{15}; }

// working-memory layout of one model with n rows, F features
struct Layout {
  uint64_t r, keys, perm, root, idx_a, idx_b, nodes, total;
  __host__ __device__ Layout(uint64_t n, uint64_t F, uint64_t max_nodes) {
    uint64_t o = 0;
    r = o;
    o = align16(o + 8 * n);
    keys = o;
    o = align16(o + 8 * F * n);
    perm = o;
    o = align16(o + 4 * F * n);
    root = o;
    o = align16(o + 4 * F * n);
    idx_a = o;
    o = align16(o + 4 * n);
    idx_b = o;
    o = align16(o + 4 * n);
    nodes = o;
    o = align16(o + sizeof(BNode) * max_nodes);
    total = o;
  }
};

__global__ void __launch_bounds__(kFitThreads) k_gbdt_fit(FitArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ double s_mean, s_lo, s_hi;
  __shared__ uint32_t s_nn, s_lvl;
  const uint32_t m = blockIdx.x;
  const uint64_t o = a.off[m];
  const uint32_t n = (uint32_t)(a.off[m + 1] - o);
  const uint32_t F = a.F, D = a.max_depth, min_leaf = a.min_leaf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* xm = a.x + o * F;  // feature f: xm + f * n
  const double* ym = a.y + o;
  double* pred = a.pred + o;
  const uint32_t max_nodes = (2u << D) - 1u;
  const Layout L(n, F, max_nodes);
  uint8_t* w = a.scratch_off[m] == ~0ull ? smem : a.scratch + a.scratch_off[m];
  double* r = (double*)(w + L.r);
  double* keys = (double*)(w + L.keys);
  uint32_t* perm = (uint32_t*)(w + L.perm);
  uint32_t* root = (uint32_t*)(w + L.root);
  uint32_t* idx = (uint32_t*)(w + L.idx_a);
  uint32_t* idx_next = (uint32_t*)(w + L.idx_b);
  BNode* nd = (BNode*)(w + L.nodes);
  cs_tree_node* out_nodes = a.nodes + (uint64_t)m * a.n_trees * a.node_stride;
  uint32_t* out_count = a.n_nodes + (uint64_t)m * a.n_trees;
  double* imp = a.importance + (uint64_t)m * F;

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
  // the root's sort permutation: same input (rows in order) for every tree
  for (uint32_t q = tid; q < F * n; q += kFitThreads) root[q] = q % n;
  __syncthreads();
  for (uint32_t f = tid; f < F; f += kFitThreads) cs_sort::sort(root + (uint64_t)f * n, n, xm + (uint64_t)f * n);
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
    for (uint32_t d = 0;; ++d) {
      const uint32_t lb = s_lvl, le = s_nn;
      if (lb == le) break;
      // (A) node totals, row order (gbdt.cpp:51-53)
      for (uint32_t j = lb + tid; j < le; j += kFitThreads) {
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        double s = 0.0;
        for (uint32_t k = 0; k < len; ++k) s += r[idx[s0 + k]];
        nd[j].sum = s;
        nd[j].feature = -1;
      }
      __syncthreads();
      auto splittable = [&](uint32_t j) { return d < D && (uint64_t)nd[j].len >= 2ull * min_leaf; };
      // (B) per feature: keys in row order and the sort permutation
      for (uint32_t j = lb; j < le; ++j) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        for (uint32_t q = tid; q < F * len; q += kFitThreads) {
          const uint32_t f = q / len, k = q - f * len;
          keys[(uint64_t)f * n + s0 + k] = xm[(uint64_t)f * n + idx[s0 + k]];
          perm[(uint64_t)f * n + s0 + k] = d == 0 ? root[(uint64_t)f * n + k] : k;
        }
      }
      __syncthreads();
      if (d > 0) {
        for (uint32_t q = tid; q < (le - lb) * F; q += kFitThreads) {
          const uint32_t j = lb + q / F, f = q % F;
          if (!splittable(j)) continue;
          const uint32_t s0 = nd[j].start;
          cs_sort::sort(perm + (uint64_t)f * n + s0, nd[j].len, keys + (uint64_t)f * n + s0);
        }
        __syncthreads();
      }
      // (C) exact greedy split, features in order with the running best (gbdt.cpp:57-90)
      for (uint32_t j = lb + tid; j < le; j += kFitThreads) {
        if (!splittable(j)) continue;
        const uint32_t s0 = nd[j].start, len = nd[j].len;
        const double sum = nd[j].sum, cnt = (double)len;
        double best_gain = 0.0, best_thr = 0.0;
        int best_f = -1;
        for (uint32_t f = 0; f < F; ++f) {
          const uint32_t* P = perm + (uint64_t)f * n + s0;
          const double* K = keys + (uint64_t)f * n + s0;
          double lsum = 0.0;
          uint32_t p = P[0];
          for (uint32_t k = 0; k + 1 < len; ++k) {
            const uint32_t pn = P[k + 1];
            lsum += r[idx[s0 + p]];
            const double kp = K[p], kn = K[pn];
            p = pn;
            if (kp == kn) continue;
            const uint32_t ln = k + 1, rn = len - ln;
            if (ln < min_leaf || rn < min_leaf) continue;
            const double rsum = sum - lsum;
            const double gain = lsum * lsum / (double)ln + rsum * rsum / (double)rn - sum * sum / cnt;
            if (gain > best_gain + 1e-12) {
              best_gain = gain;
              best_f = (int)f;
              best_thr = 0.5 * (kp + kn);
            }
          }
        }
        if (best_f >= 0 && best_gain > 1e-12) {
          nd[j].feature = best_f;
          nd[j].thr = best_thr;
          nd[j].gain = best_gain;
        }
      }
      __syncthreads();
      // (D) stable split of each internal node's rows (gbdt.cpp:97-104), warp per node
      for (uint32_t j = lb + warp; j < le; j += kFitThreads / 32) {
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
  DevMem d_off, d_x, d_y, d_pred, d_scr, d_scr_off, d_nodes, d_cnt, d_base, d_deg, d_imp;
  auto alloc = [&](DevMem& x, size_t bytes) { return cudaMalloc(&x.p, std::max<size_t>(bytes, 16)) == cudaSuccess; };
  const size_t node_count = static_cast<size_t>(M) * b.params.n_trees * max_nodes;
  if (!alloc(d_off, (M + 1) * 8) || !alloc(d_x, rows * F * 8) || !alloc(d_y, rows * 8) ||
      !alloc(d_pred, rows * 8) || !alloc(d_scr, scratch_total) || !alloc(d_scr_off, M * 8) ||
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
  a.pred = static_cast<double*>(d_pred.p);
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
