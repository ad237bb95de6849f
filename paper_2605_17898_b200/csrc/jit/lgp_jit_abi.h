// Argument blocks shared by the host launcher (lgp_*.cpp, compiled by nvcc/g++)
// and the NVRTC-generated kernels (this text is prepended to every JIT source).
// Plain C layout only: both sides must agree byte for byte.
#ifndef LGP_JIT_ABI_H_
#define LGP_JIT_ABI_H_

#define LGP_MAX_KC 48
#define LGP_MAX_PC 48

// Per-point feature preparation: x (FP64, n x d) -> row / column features (FP32).
struct LgpPrepArgs {
  const double* x;      // points, n x d row-major
  const double* ctr;    // d centring offsets (column mean of the column set)
  float* fr;            // [n_pad][FR] row-side features (may be null)
  float* fc;            // [n_pad][FC] column-side features (may be null)
  float* f32;           // tensor-core prep: [n_pad][FW] FP32 features (may be null)
  long long row0;       // first point to prepare (sharded row slice)
  long long n;          // points in this slice
  long long n_pad;      // padded slice length (zero features beyond n)
  double pc[LGP_MAX_PC];
};

// Fused matrix-free K·V: one CTA = (row block, column segment, RHS pass).
struct LgpMatvecArgs {
  const float* fr;      // [n_rows_pad][FR]
  const float* fc;      // [n_cols_pad][FC]
  const double* v;      // packed RHS [n_pass][n_cols_pad][TB]
  double* partial;      // [n_seg][n_pass][n_rows_pad][TB]
  const int* done;      // optional early-exit flag (solver loops), may be null
  int n_rows_pad;
  int n_cols_pad;
  int n_rb;             // row blocks
  int n_seg;            // column segments
  int n_pass;           // RHS passes of TB columns
  int tiles_per_seg;
  int n_tiles;          // column tiles in total
  int n_units;          // symmetric kernel: block pairs (I, J >= I)
  const int* units;     // symmetric kernel: [n_units][2] = (I, J)
  double* colpart;      // symmetric kernel: column-side partials, like partial
  float kc[LGP_MAX_KC];
};

// Dense FP64 cross-covariance / diagonal.
struct LgpGramArgs {
  const double* x;      // rows, n_rows x d
  const double* y;      // cols, n_cols x d
  double* out;          // n_rows x ld
  long long n_rows;
  long long n_cols;
  long long ld;
  double pc[LGP_MAX_PC];
};

#endif  // LGP_JIT_ABI_H_

#ifndef LGP_TC_ABI_
#define LGP_TC_ABI_
// Tensor-core K1 (tcgen05, kind::f16): operands are pre-tiled in the UMMA
// K-major no-swizzle canonical layout by the prep / pack kernels.
struct LgpTcArgs {
  const float* a1;      // row operand tiles (FP16 hi/lo features) [n_rb][128 x KD]
  const float* b1;      // column operand tiles [n_tiles][64 x KD]
  const float* r32;     // FP32 row features [n_rows_pad][FW] = (c_i, -|c_i|^2, 0..)
  const float* c32;     // FP32 column features [n_cols_pad][FW] = (2 c_j, -|c_j|^2, 0..)
  const void* v;        // RHS tiles (FP16 hi/lo) [n_pass][n_tiles][2][TBN x 64]
  const float* vscale;  // power-of-two scale of each RHS column [n_pass * TBN]
  double* partial;      // [n_seg][n_pass][n_rows_pad][TBN]
  const int* done;      // optional early-exit flag
  const int* v_inexact; // set by the RHS pack kernel if any V_lo != 0 (may be null)
  unsigned long long* trace;  // LGP_TC_TRACE builds only: cycle counters
  int n_rows_pad;
  int n_rb;
  int n_seg;
  int n_pass;
  int tiles_per_seg;
  int n_tiles;
  int seg_base;         // first column segment of this launch (staged uploads: one launch per part)
  int seg_split;        // segments >= seg_split scale V by the second half of vscale (two parts)
  float kc[LGP_MAX_KC];
};

// Symmetric tensor-core K1 for the square operator with one RHS (the CG
// matvec): every unordered pair (i, j) is evaluated once, in the tile of row
// block min and column chunk max, and feeds out_i and out_j in FP64. Work
// item = rectangle of row blocks [Ia, Ib) x 64-column chunks [ca, cb), at
// most R x 2R.
struct LgpTcSymArgs {
  const float* a1;            // row operand tiles (FP16 hi/lo features) [n_rb][128 x KD]
  const float* b1;            // column operand tiles [n_tiles][64 x KD]
  const double* v;            // RHS, zero-padded to the column padding (t = 1)
  const float* r32;           // FP32 row features [n_rows_pad][FW] (Periodic trees; else null)
  const float* c32;           // FP32 column features [n_cols_pad][FW] (Periodic trees; else null)
  const int* items;           // [n_items][6]: (Ia, Ib, ca, cb, first row record, first chunk record)
  double* rowpart;            // [row records of the launched items][128]
  double* colpart;            // [chunk records of the launched items][64]
  const int* done;            // optional early-exit flag
  int item_base;              // first work item of this launch (multi-rank CG: the rank's share)
  int R;                      // max row blocks per item (column accumulators: 2R x 64)
  int n_rb;                   // row blocks (128 rows)
  int n_tiles;                // 64-column chunks
  float kc[LGP_MAX_KC];
};
#endif
