// HODLRdD operator on the device: batched dense leaf / near-field block assembly and the
// hierarchical matvec (hmatrix.hpp:50-179, cluster_tree.hpp:107-229).
//
// Host (this file, restating cluster_tree.hpp): the balanced 2^d tree over the domain cube
// (stable counting split of every box until all hold <= n_max points; points on an internal
// face go to the lower box) and the block structure of an admissibility policy (candidate pairs
// = siblings + children of the parent's deferred pairs; admissible ones are compressed at that
// level, the rest recurse and end as dense leaf pairs).
// Device:
//   * all dense blocks — leaf self blocks and the near field — assembled by ONE launch of
//     block_assemble_kernel (32 x 32 tiles of every block, block found by binary search over the
//     tile prefix), entries by the k2 rule (entries.cuh, r bit-identical to assemble_dense);
//   * every admissible block compressed by the device ACA (aca.cu, batched: one launch for all
//     blocks that fit one CTA);
//   * matvec b = K q: gather q into tree order; per low-rank block t = U⁻¹ L⁻¹ K(σ, J) q_J (one
//     CTA per block, entries recomputed on the fly, aca.hpp:202-213); per level y_I += K(I, τ) t
//     (one thread per row, blocks of the row's box in the reference's pair order); dense rows
//     y_I += K_blk q_J (self block, then the near field); scatter back to the original order.
//     No atomics: every row's sum has a fixed order, so matvecs are bit-reproducible.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <vector>

#include "context.h"
#include "entries.cuh"
#include "hmatrix.h"

namespace hb {

namespace {

DevKernel devk(const hb_kernel& k) {
  DevKernel K;
  K.id = k.id;
  K.has_diag = k.has_diag != 0;
  K.diag = k.diag;
  K.singular = kernel_singular_at_origin(k.id) ? 1 : 0;
  return K;
}

// ---- host tree (cluster_tree.hpp:180-229, geometry.hpp:121-151) -------------------------------
std::vector<int> box_grid(int d, int level, int64_t id) {
  std::vector<int> g(d, 0);
  for (int lev = level - 1; lev >= 0; --lev) {
    const uint64_t c = ((uint64_t)id >> (d * lev)) & ((1ull << d) - 1ull);
    for (int k = 0; k < d; ++k) g[k] = (g[k] << 1) | (int)((c >> k) & 1u);
  }
  return g;
}

// classify_pair (geometry.hpp:109-118): 0 self, 1 surface (dp = #zero offsets), 2 far
int classify(const std::vector<int>& a, const std::vector<int>& b, int* dp) {
  bool zero = true;
  int mx = 0, zeros = 0;
  for (size_t k = 0; k < a.size(); ++k) {
    const int o = std::abs(a[k] - b[k]);
    zero &= o == 0;
    mx = std::max(mx, o);
    zeros += o == 0;
  }
  *dp = zeros;
  if (zero) return 0;
  if (mx >= 2) return 2;
  return 1;
}

// is_admissible (cluster_tree.hpp:22-29): WeakDD far|vertex, Strong far, WeakAll non-self
bool admissible(int policy, int cls, int dp) {
  if (policy == HB_POLICY_WEAKDD) return cls == 2 || (cls == 1 && dp == 0);
  if (policy == HB_POLICY_STRONG) return cls == 2;
  return cls != 0;
}

void build_tree(hb_hmatrix& h, const double* P, const hb_cube& dom, int64_t n_max) {
  const int d = h.d;
  const int64_t n = h.N;
  std::vector<int64_t> perm((size_t)n);
  std::iota(perm.begin(), perm.end(), 0);
  h.nb.assign(1, {0});
  h.ne.assign(1, {n});
  const int64_t nch = 1ll << d;
  int depth = 0;
  for (;;) {
    bool fits = true;
    for (size_t b = 0; b < h.nb[depth].size(); ++b)
      if (h.ne[depth][b] - h.nb[depth][b] > n_max) { fits = false; break; }
    if (fits) break;
    if ((depth + 1) * d > 60 || depth >= 40)
      throw Error(HB_ECAP, "build_tree: subdivision limit reached (coincident points?)");
    const int64_t nodes = 1ll << (d * (depth + 1));
    std::vector<int64_t> nbeg((size_t)nodes), nend((size_t)nodes);
    std::vector<int64_t> scratch(perm.size());
    const double hside = dom.side / (double)(1ll << depth);  // box_cube (geometry.hpp:146-151)
    for (int64_t b = 0; b < (int64_t)h.nb[depth].size(); ++b) {
      const int64_t b0 = h.nb[depth][(size_t)b], b1 = h.ne[depth][(size_t)b];
      const std::vector<int> g = box_grid(d, depth, b);
      double c[8];
      for (int k = 0; k < d; ++k) {
        const double lo = dom.lower[k] + hside * g[k];
        c[k] = lo + 0.5 * hside;  // HyperCube::center
      }
      auto child_of = [&](int64_t p) {
        uint64_t cc = 0;
        for (int k = 0; k < d; ++k)
          if (P[(int64_t)k * n + p] > c[k]) cc |= (1ull << k);
        return (int64_t)cc;
      };
      std::vector<int64_t> count((size_t)nch, 0), offset((size_t)nch, 0);
      for (int64_t t = b0; t < b1; ++t) ++count[(size_t)child_of(perm[(size_t)t])];
      int64_t acc = b0;
      for (int64_t cc = 0; cc < nch; ++cc) {
        offset[(size_t)cc] = acc;
        nbeg[(size_t)(b * nch + cc)] = acc;
        acc += count[(size_t)cc];
        nend[(size_t)(b * nch + cc)] = acc;
      }
      for (int64_t t = b0; t < b1; ++t) scratch[(size_t)offset[(size_t)child_of(perm[(size_t)t])]++] = perm[(size_t)t];
      std::copy(scratch.begin() + b0, scratch.begin() + b1, perm.begin() + b0);
    }
    h.nb.push_back(std::move(nbeg));
    h.ne.push_back(std::move(nend));
    ++depth;
  }
  h.depth = depth;
  h.orig_of_tree = perm;
}

struct Blocks {
  std::vector<std::vector<std::pair<int64_t, int64_t>>> adm;  // per level
  std::vector<std::pair<int64_t, int64_t>> near;
};

// block_structure (cluster_tree.hpp:107-137)
Blocks block_structure(const hb_hmatrix& h, int policy) {
  const int d = h.d;
  Blocks bs;
  bs.adm.resize((size_t)h.depth + 1);
  std::vector<std::vector<int64_t>> deferred(1);
  for (int level = 1; level <= h.depth; ++level) {
    const int64_t nodes = 1ll << (d * level);
    std::vector<std::vector<int64_t>> next((size_t)nodes);
    const int64_t nch = 1ll << d;
    for (int64_t i = 0; i < nodes; ++i) {
      const int64_t parent = i >> d;
      const std::vector<int> bi = box_grid(d, level, i);
      auto consider = [&](int64_t j) {
        if (j == i) return;
        int dp = 0;
        const int cls = classify(bi, box_grid(d, level, j), &dp);
        if (admissible(policy, cls, dp)) bs.adm[(size_t)level].emplace_back(i, j);
        else next[(size_t)i].push_back(j);
      };
      for (int64_t c = 0; c < nch; ++c) consider(parent * nch + c);
      for (int64_t p : deferred[(size_t)parent])
        for (int64_t c = 0; c < nch; ++c) consider(p * nch + c);
      std::sort(next[(size_t)i].begin(), next[(size_t)i].end());
    }
    deferred = std::move(next);
  }
  for (int64_t i = 0; i < (int64_t)deferred.size(); ++i)
    for (int64_t j : deferred[(size_t)i]) bs.near.emplace_back(i, j);
  return bs;
}

// ---- device kernels ------------------------------------------------------------------------
constexpr int kTile = 32;

// every dense block in 32 x 32 tiles; tile_first[b] = first tile of block b (prefix, nb + 1)
__global__ void block_assemble_kernel(DevKernel K, int d, const double* __restrict__ pts, int64_t n,
                                      const int64_t* __restrict__ desc, const int64_t* __restrict__ tile_first,
                                      int64_t nblk, double* __restrict__ out, unsigned int* flags) {
  const int64_t tile = blockIdx.x;
  int64_t lo = 0, hi = nblk - 1;
  while (lo < hi) {  // last b with tile_first[b] <= tile
    const int64_t mid = (lo + hi + 1) >> 1;
    if (tile_first[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const int64_t b = lo;
  const int64_t rb = desc[5 * b], rows = desc[5 * b + 1], cb = desc[5 * b + 2], cols = desc[5 * b + 3],
                off = desc[5 * b + 4];
  const int64_t tr = ceil_div(rows, kTile);
  const int64_t t = tile - tile_first[b];
  const int64_t r0 = (t % tr) * kTile, c0 = (t / tr) * kTile;
  unsigned int bad = 0;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int64_t r = r0 + (e % kTile), c = c0 + (e / kTile);
    if (r < rows && c < cols) out[off + r + c * rows] = entry_soa(K, pts, n, rb + r, pts, n, cb + c, d, &bad);
  }
  if (bad) atomicOr(flags, bad);
}

__global__ void gather_kernel(const double* __restrict__ q, const int64_t* __restrict__ orig, int64_t n,
                              double* __restrict__ qt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) qt[t] = q[orig[t]];
}

__global__ void scatter_kernel(const double* __restrict__ yt, const int64_t* __restrict__ orig, int64_t n,
                               double* __restrict__ b) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) b[orig[t]] = yt[t];
}

// t = U⁻¹ L⁻¹ K(σ, J) q_J for one low-rank block per CTA (aca.hpp:206-209)
__global__ void lr_rows_kernel(DevKernel K, int d, const double* __restrict__ pts, int64_t n,
                               const int64_t* __restrict__ desc, const int64_t* __restrict__ piv,
                               const double* __restrict__ lu, const double* __restrict__ qt,
                               double* __restrict__ tv, unsigned int* flags) {
  __shared__ double red[32];
  const int64_t* D = desc + 8 * blockIdx.x;
  const int64_t cb = D[2], cols = D[3], r = D[4], po = D[5], to = D[6], lo = D[7];
  double* t = tv + to;
  unsigned int bad = 0;
  for (int64_t k = 0; k < r; ++k) {
    const int64_t i = piv[po + k];
    double a = 0.0;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
      a += entry_soa(K, pts, n, i, pts, n, cb + j, d, &bad) * qt[cb + j];
    a = block_sum(a, red);
    if (threadIdx.x == 0) t[k] = a;
  }
  const double* L = lu + lo;
  const double* U = L + r * r;
  for (int64_t k = 0; k < r; ++k) {  // unit lower, column-oriented (the reference's order)
    __syncthreads();
    const double tk = t[k];
    for (int64_t i = k + 1 + threadIdx.x; i < r; i += blockDim.x)
      t[i] = __dsub_rn(t[i], __dmul_rn(L[i + k * r], tk));
  }
  for (int64_t k = r - 1; k >= 0; --k) {  // upper
    __syncthreads();
    const double tk = __ddiv_rn(t[k], U[k + k * r]);
    __syncthreads();
    if (threadIdx.x == 0) t[k] = tk;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x)
      t[i] = __dsub_rn(t[i], __dmul_rn(U[i + k * r], tk));
  }
  if (bad) atomicOr(flags, bad);
}

// one level: y_t += Σ_blocks of t's box (pair order) Σ_k t_k K(t, τ_k)   (aca.hpp:210-211)
__global__ void lr_cols_kernel(DevKernel K, int d, const double* __restrict__ pts, int64_t n,
                               const int64_t* __restrict__ desc, const int64_t* __restrict__ piv,
                               const double* __restrict__ tv, const int64_t* __restrict__ box_begin,
                               const int64_t* __restrict__ box_first, int64_t nboxes, int64_t lr0,
                               double* __restrict__ y, unsigned int* flags) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= n) return;
  int64_t lo = 0, hi = nboxes - 1;
  while (lo < hi) {  // box containing row: last box with begin <= row (empty boxes share begins)
    const int64_t mid = (lo + hi + 1) >> 1;
    if (box_begin[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  unsigned int bad = 0;
  double yv = y[row];
  for (int64_t bi = box_first[lo]; bi < box_first[lo + 1]; ++bi) {
    const int64_t* D = desc + 8 * (lr0 + bi);
    const int64_t rb = D[0], rows = D[1], r = D[4], po = D[5], to = D[6];
    if (row < rb || row >= rb + rows || r == 0) continue;
    double acc = 0.0;
    for (int64_t k = 0; k < r; ++k)
      acc = __dadd_rn(acc, __dmul_rn(tv[to + k], entry_soa(K, pts, n, row, pts, n, piv[po + r + k], d, &bad)));
    yv = __dadd_rn(yv, acc);
  }
  y[row] = yv;
  if (bad) atomicOr(flags, bad);
}

// dense rows: y_t += Σ_{dense blocks of t's leaf} K_blk(t - rb, :) q_J
__global__ void dense_rows_kernel(const int64_t* __restrict__ desc, const int64_t* __restrict__ leaf_first,
                                  const int64_t* __restrict__ leaf_begin, int64_t nleaves,
                                  const double* __restrict__ vals, const double* __restrict__ qt, int64_t n,
                                  double* __restrict__ y) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= n) return;
  int64_t lo = 0, hi = nleaves - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (leaf_begin[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  double yv = y[row];
  for (int64_t b = leaf_first[lo]; b < leaf_first[lo + 1]; ++b) {
    const int64_t rb = desc[5 * b], rows = desc[5 * b + 1], cb = desc[5 * b + 2], cols = desc[5 * b + 3],
                  off = desc[5 * b + 4];
    if (row < rb || row >= rb + rows) continue;
    const double* Kb = vals + off + (row - rb);
    double acc = 0.0;
    for (int64_t c = 0; c < cols; ++c) acc = __dadd_rn(acc, __dmul_rn(Kb[c * rows], qt[cb + c]));
    yv = __dadd_rn(yv, acc);
  }
  y[row] = yv;
}

template <typename T>
T* upload(const std::vector<T>& v, cudaStream_t st) {
  void* p = nullptr;
  HB_CUDA(cudaMallocAsync(&p, std::max<size_t>(v.size(), 1) * sizeof(T), st));
  if (!v.empty()) HB_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return static_cast<T*>(p);
}

}  // namespace

void hmatrix_free(hb_hmatrix* h) {
  // synchronous frees, independent of the context: an operator may outlive its context (a Python
  // finaliser running after the context was closed) and must still release cleanly
  if (!h) return;
  if (h->device >= 0) cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (void* p : {(void*)h->pts, (void*)h->d_orig, (void*)h->d_dense, (void*)h->d_leaf_first,
                  (void*)h->d_leaf_begin, (void*)h->dense_vals, (void*)h->d_lr, (void*)h->d_piv,
                  (void*)h->d_lu, (void*)h->d_t, (void*)h->d_y, (void*)h->d_q, (void*)h->d_flags})
    if (p) cudaFree(p);
  for (auto* p : h->d_box_first) if (p) cudaFree(p);
  for (auto* p : h->d_box_begin) if (p) cudaFree(p);
  for (auto& b : h->lr)
    if (b.f) hb_aca_factor_destroy(b.f);
  h->lr.clear();
}

void hmatrix_build(hb_hmatrix* h, const double* P, const hb_cube& dom, int64_t n_max, double eps,
                   int64_t max_rank, int64_t dense_cap) {
  const auto t0 = std::chrono::steady_clock::now();
  hb_context* c = h->ctx;
  cudaStream_t st = c->stream;
  const int d = h->d;
  const int64_t n = h->N;
  build_tree(*h, P, dom, n_max);
  const Blocks bs = block_structure(*h, h->policy);
  const int depth = h->depth;
  const int64_t nleaves = 1ll << (d * depth);
  auto sz = [&](int lv, int64_t i) { return h->ne[(size_t)lv][(size_t)i] - h->nb[(size_t)lv][(size_t)i]; };
  // dense storage first so the entry cap fails fast (hmatrix.hpp:71-79)
  int64_t dense_entries = 0;
  for (int64_t i = 0; i < nleaves; ++i) dense_entries += sz(depth, i) * sz(depth, i);
  for (const auto& pr : bs.near) dense_entries += sz(depth, pr.first) * sz(depth, pr.second);
  if (dense_entries > dense_cap) throw Error(HB_ECAP, "HMatrix: dense leaf storage exceeds the entry cap");
  h->dense_entries = dense_entries;
  // dense blocks grouped by row leaf: self, then near pairs (bs.near is by i, j ascending)
  std::vector<int64_t> leaf_first((size_t)nleaves + 1, 0), leaf_begin((size_t)nleaves + 1, 0);
  {
    size_t q = 0;
    int64_t off = 0;
    for (int64_t i = 0; i < nleaves; ++i) {
      leaf_first[(size_t)i] = (int64_t)h->dense.size();
      leaf_begin[(size_t)i] = h->nb[(size_t)depth][(size_t)i];
      if (sz(depth, i) > 0) {
        h->dense.push_back({h->nb[(size_t)depth][(size_t)i], sz(depth, i), h->nb[(size_t)depth][(size_t)i], sz(depth, i), off});
        off += sz(depth, i) * sz(depth, i);
      }
      for (; q < bs.near.size() && bs.near[q].first == i; ++q) {
        const int64_t j = bs.near[q].second;
        if (sz(depth, i) == 0 || sz(depth, j) == 0) continue;
        h->dense.push_back({h->nb[(size_t)depth][(size_t)i], sz(depth, i), h->nb[(size_t)depth][(size_t)j], sz(depth, j), off});
        off += sz(depth, i) * sz(depth, j);
      }
    }
    leaf_first[(size_t)nleaves] = (int64_t)h->dense.size();
    leaf_begin[(size_t)nleaves] = n;
  }
  // points in tree order on the device
  std::vector<double> pt((size_t)(d * n));
  for (int64_t t = 0; t < n; ++t)
    for (int k = 0; k < d; ++k) pt[(size_t)(k * n + t)] = P[(int64_t)k * n + h->orig_of_tree[(size_t)t]];
  h->pts = upload(pt, st);
  h->d_orig = upload(h->orig_of_tree, st);
  HB_CUDA(cudaMallocAsync((void**)&h->d_flags, sizeof(unsigned int), st));
  HB_CUDA(cudaMemsetAsync(h->d_flags, 0, sizeof(unsigned int), st));
  const DevKernel K = devk(h->kern);
  {
    std::vector<int64_t> desc, tile_first;
    int64_t tiles = 0;
    for (const auto& b : h->dense) {
      desc.insert(desc.end(), {b.rb, b.rows, b.cb, b.cols, b.off});
      tile_first.push_back(tiles);
      tiles += ceil_div(b.rows, kTile) * ceil_div(b.cols, kTile);
    }
    tile_first.push_back(tiles);
    h->d_dense = upload(desc, st);
    h->d_leaf_first = upload(leaf_first, st);
    h->d_leaf_begin = upload(leaf_begin, st);
    HB_CUDA(cudaMallocAsync((void**)&h->dense_vals, sizeof(double) * std::max<int64_t>(dense_entries, 1), st));
    int64_t* d_tf = upload(tile_first, st);
    if (tiles > 0) {
      HB_REQUIRE(tiles < (1ll << 31), HB_ECAP, "HMatrix: too many dense tiles");
      block_assemble_kernel<<<(unsigned)tiles, 256, 0, st>>>(K, d, h->pts, n, h->d_dense, d_tf,
                                                             (int64_t)h->dense.size(), h->dense_vals, h->d_flags);
      HB_LAUNCH_CHECK();
    }
    HB_CUDA(cudaFreeAsync(d_tf, st));
  }
  // admissible blocks, level by level in the reference's pair order; ACA on all non-empty ones
  // in one batched call
  std::vector<hb_block> blks;
  std::vector<size_t> which;
  h->lvl_first.assign((size_t)depth + 2, 0);
  for (int level = 1; level <= depth; ++level) {
    h->lvl_first[(size_t)level] = (int64_t)h->lr.size();
    for (const auto& pr : bs.adm[(size_t)level]) {
      hb_hmatrix::LR b{level, pr.first, pr.second, h->nb[(size_t)level][(size_t)pr.first], sz(level, pr.first),
                       h->nb[(size_t)level][(size_t)pr.second], sz(level, pr.second), nullptr};
      if (b.rows > 0 && b.cols > 0) {
        blks.push_back(hb_block{b.rb, b.rows, b.cb, b.cols});
        which.push_back(h->lr.size());
      }
      h->lr.push_back(b);
    }
  }
  h->lvl_first[(size_t)depth + 1] = (int64_t)h->lr.size();
  if (!blks.empty()) {
    std::vector<hb_aca_factor*> fs(blks.size(), nullptr);
    aca_compress(c, h->kern, h->pts, n, h->pts, n, d, blks.data(), (int64_t)blks.size(), eps, max_rank, fs.data());
    for (size_t q = 0; q < fs.size(); ++q) h->lr[which[q]].f = fs[q];
  }
  // device descriptors of the low-rank blocks: rb rows cb cols rank piv_off t_off lu_off
  std::vector<int64_t> desc, piv;
  std::vector<double> lu;
  int64_t toff = 0;
  hb_build_report& rep = h->report;
  rep = hb_build_report{};
  for (auto& b : h->lr) {
    const int64_t r = b.f ? b.f->rank : 0;
    desc.insert(desc.end(), {b.rb, b.rows, b.cb, b.cols, r, (int64_t)piv.size(), toff, (int64_t)lu.size()});
    if (r > 0) {
      piv.insert(piv.end(), b.f->sigma.begin(), b.f->sigma.end());
      piv.insert(piv.end(), b.f->tau.begin(), b.f->tau.end());
      std::vector<double> Lh((size_t)(r * r)), Uh((size_t)(r * r));
      HB_CUDA(cudaMemcpy(Lh.data(), b.f->L, sizeof(double) * r * r, cudaMemcpyDeviceToHost));
      HB_CUDA(cudaMemcpy(Uh.data(), b.f->U, sizeof(double) * r * r, cudaMemcpyDeviceToHost));
      lu.insert(lu.end(), Lh.begin(), Lh.end());
      lu.insert(lu.end(), Uh.begin(), Uh.end());
    }
    toff += r;
    // BuildReport (hmatrix.hpp:111-122)
    ++rep.num_low_rank_blocks;
    rep.max_block_rank = std::max<int32_t>(rep.max_block_rank, (int32_t)r);
    if (b.f && !b.f->met) ++rep.num_tolerance_failures;
    rep.memory_bytes += 2 * r * r * (int64_t)sizeof(double) + 2 * r * (int64_t)sizeof(int64_t);
  }
  h->t_total = toff;
  h->d_lr = upload(desc, st);
  h->d_piv = upload(piv, st);
  h->d_lu = upload(lu, st);
  for (int level = 0; level <= depth; ++level) {  // per level CSR over boxes (pairs sorted by i)
    const int64_t nodes = 1ll << (d * level);
    std::vector<int64_t> first((size_t)nodes + 1, 0), beg((size_t)nodes + 1, n);
    const int64_t l0 = level >= 1 ? h->lvl_first[(size_t)level] : 0;
    const int64_t l1 = level >= 1 ? h->lvl_first[(size_t)level + 1] : 0;
    int64_t q = l0;
    for (int64_t i = 0; i < nodes; ++i) {
      first[(size_t)i] = q - l0;
      beg[(size_t)i] = h->nb[(size_t)level][(size_t)i];
      while (q < l1 && h->lr[(size_t)q].i == i) ++q;
    }
    first[(size_t)nodes] = q - l0;
    h->d_box_first.push_back(upload(first, st));
    h->d_box_begin.push_back(upload(beg, st));
  }
  HB_CUDA(cudaMallocAsync((void**)&h->d_t, sizeof(double) * std::max<int64_t>(toff, 1), st));
  HB_CUDA(cudaMallocAsync((void**)&h->d_y, sizeof(double) * n, st));
  HB_CUDA(cudaMallocAsync((void**)&h->d_q, sizeof(double) * n, st));
  unsigned int f = 0;
  HB_CUDA(cudaMemcpyAsync(&f, h->d_flags, sizeof(f), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  if (f & 1u) throw Error(HB_ESINGULAR, "kernel eval: r == 0 on a singular kernel with no diagonal value");
  rep.num_dense_entries = dense_entries;
  rep.memory_bytes += dense_entries * (int64_t)sizeof(double);
  rep.depth = depth;
  rep.init_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void hmatrix_matvec(hb_hmatrix* h, const double* d_q, double* d_b) {
  hb_context* c = h->ctx;
  cudaStream_t st = c->stream;
  const int64_t n = h->N;
  const int d = h->d;
  const DevKernel K = devk(h->kern);
  const unsigned g = (unsigned)ceil_div(n, 256);
  gather_kernel<<<g, 256, 0, st>>>(d_q, h->d_orig, n, h->d_q);
  HB_CUDA(cudaMemsetAsync(h->d_y, 0, sizeof(double) * n, st));
  const int64_t nlr = (int64_t)h->lr.size();
  if (nlr > 0) {
    lr_rows_kernel<<<(unsigned)nlr, 256, 0, st>>>(K, d, h->pts, n, h->d_lr, h->d_piv, h->d_lu, h->d_q, h->d_t,
                                                  h->d_flags);
    HB_LAUNCH_CHECK();
    for (int level = 1; level <= h->depth; ++level) {
      const int64_t l0 = h->lvl_first[(size_t)level];
      if (h->lvl_first[(size_t)level + 1] == l0) continue;
      lr_cols_kernel<<<g, 256, 0, st>>>(K, d, h->pts, n, h->d_lr, h->d_piv, h->d_t, h->d_box_begin[(size_t)level],
                                        h->d_box_first[(size_t)level], 1ll << (d * level), l0, h->d_y, h->d_flags);
      HB_LAUNCH_CHECK();
    }
  }
  dense_rows_kernel<<<g, 256, 0, st>>>(h->d_dense, h->d_leaf_first, h->d_leaf_begin, 1ll << (d * h->depth),
                                       h->dense_vals, h->d_q, n, h->d_y);
  scatter_kernel<<<g, 256, 0, st>>>(h->d_y, h->d_orig, n, d_b);
  HB_LAUNCH_CHECK();
}

}  // namespace hb
