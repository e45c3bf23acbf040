// hb_hmatrix: the device HODLRdD operator (hmatrix.cu) behind the opaque ABI handle.
#pragma once

#include <cstdint>
#include <vector>

#include "hb.h"

struct hb_context;
struct hb_aca_factor;

struct hb_hmatrix {
  hb_context* ctx = nullptr;
  int device = -1;
  hb_kernel kern{};
  int d = 0, depth = 0, policy = 0;
  int64_t N = 0;
  std::vector<int64_t> orig_of_tree;
  std::vector<std::vector<int64_t>> nb, ne;  // node ranges [begin, end) per level
  double* pts = nullptr;      // tree-ordered points, SoA
  int64_t* d_orig = nullptr;  // tree id -> original id
  // dense blocks, grouped by row leaf (self first, then near pairs in the reference's order)
  struct Dense { int64_t rb, rows, cb, cols, off; };
  std::vector<Dense> dense;
  int64_t* d_dense = nullptr;      // [5 * ndense]
  int64_t* d_leaf_first = nullptr; // [n_leaves + 1] CSR over dense blocks by row leaf
  int64_t* d_leaf_begin = nullptr; // [n_leaves + 1] row begin of each leaf (+ N)
  double* dense_vals = nullptr;
  int64_t dense_entries = 0;
  // low-rank blocks per level
  struct LR { int level; int64_t i, j, rb, rows, cb, cols; hb_aca_factor* f; };
  std::vector<LR> lr;
  int64_t* d_lr = nullptr;        // [8 * nlr] rb rows cb cols rank piv_off t_off lu_off
  int64_t* d_piv = nullptr;       // sigma then tau per block
  double* d_lu = nullptr;         // L then U per block (rank^2 each)
  std::vector<int64_t> lvl_first; // lr index range per level (blocks sorted by level)
  std::vector<int64_t*> d_box_first;  // per level CSR [boxes + 1] over that level's lr blocks
  std::vector<int64_t*> d_box_begin;  // per level node begins [boxes + 1]
  int64_t t_total = 0;
  double* d_t = nullptr;
  double* d_y = nullptr;
  double* d_q = nullptr;
  unsigned int* d_flags = nullptr;
  hb_build_report report{};
};
