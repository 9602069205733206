// Lazy TT expressions: device-side descriptors and evaluator.
//
// A (pre-rounding) TT is a list of terms; each term is a rank-r_t pair of core
// expressions (X side m x r_t, Yt side n x r_t). A core expression is a base panel
// followed by a chain of one-mode operations: scalings (tt.hpp:163-166) and banded maps
// (apply_core_map, tt.hpp:185-194, with the operators of reconstruction.hpp:428-501).
// Term kinds: plain base cores; Hadamard (face-splitting, tt.hpp:169-181) of two
// materialised operands; constant rank-1 (TTMatrix::zero/constant, tt.hpp:35-41).
//
// Evaluation reproduces the op-by-op arithmetic exactly: every intermediate element is
// the same sum of products in the same order as when the maps are applied one after
// the other, so the gathered panels equal what the materialising path would write.
#pragma once

#include "ttsw.hpp"

namespace ttsw {

constexpr int kMaxSideOps = 10;

/// POD copy of BandMap for device code.
struct MapDesc {
  long n_out, n_in;
  int period, stride, taps, wrap;
  int off[3];
  double coef[3][5];
};

struct SideOp {
  int kind;  // 0 = scale, 1 = map
  int map;   // index into the context's map table
  double scale;
};

struct SideExpr {
  const double* base;
  long ld;
  int nops;
  SideOp ops[kMaxSideOps];
};

enum TermKind : int { TERM_PLAIN = 0, TERM_HADAMARD = 1, TERM_CONST = 2 };

struct TermDesc {
  int kind;
  int r;        // columns contributed by the term
  long col0;    // first output column
  SideExpr x, y;            // PLAIN: bases; HADAMARD: first operand (rank r / r2)
  const double* x2;         // HADAMARD second operand X (ld = ldx2)
  const double* y2;         // HADAMARD second operand Yt (ld = ldy2)
  long ldx2, ldy2;
  int r2;
  double cx, cy;            // CONST: core_x value, core_y value
};

#ifdef __CUDACC__
__device__ inline double term_base(const TermDesc& t, int side, long row, int c) {
  if (t.kind == TERM_CONST) return side == 0 ? t.cx : t.cy;
  const SideExpr& s = side == 0 ? t.x : t.y;
  if (t.kind == TERM_HADAMARD) {
    const int a = c / t.r2, b = c % t.r2;
    const double v2 = side == 0 ? t.x2[row + long(b) * t.ldx2] : t.y2[row + long(b) * t.ldy2];
    return v2 * s.base[row + long(a) * s.ld];  // y.cx(i,b) * x.cx(i,a)
  }
  return s.base[row + long(c) * s.ld];
}

/// Value at `row` after the first k ops of the side chain (recursive over maps).
__device__ inline double eval_side(const TermDesc& t, int side, const MapDesc* maps, int k, long row, int c) {
  const SideExpr& s = side == 0 ? t.x : t.y;
  // peel trailing scalings iteratively
  double mul_chain[kMaxSideOps];
  int nscale = 0;
  while (k > 0 && s.ops[k - 1].kind == 0) {
    mul_chain[nscale++] = s.ops[k - 1].scale;
    --k;
  }
  double v;
  if (k == 0) {
    v = term_base(t, side, row, c);
  } else {
    const MapDesc& m = maps[s.ops[k - 1].map];
    const int ph = int(row % m.period);
    const long base = (row / m.period) * m.stride + m.off[ph];
    double acc = 0.0;
    for (int tp = 0; tp < m.taps; ++tp) {
      long r2 = base + tp;
      if (m.wrap) {  // periodic pad: offsets are within one period
        if (r2 < 0) r2 += m.n_in;
        else if (r2 >= m.n_in) r2 -= m.n_in;
      }
      acc += m.coef[ph][tp] * eval_side(t, side, maps, k - 1, r2, c);
    }
    v = acc;
  }
  for (int q = nscale - 1; q >= 0; --q) v = v * mul_chain[q];
  return v;
}

/// Locate the term owning output column `col` (terms sorted by col0).
__device__ inline int find_term(const TermDesc* terms, int nterms, long col) {
  int lo = 0, hi = nterms - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (terms[mid].col0 <= col) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

/// Element (row, col) of side `side` of the whole expression.
__device__ inline double expr_value(const TermDesc* terms, int nterms, const MapDesc* maps, int side, long row,
                                    long col) {
  const TermDesc& t = terms[find_term(terms, nterms, col)];
  const SideExpr& s = side == 0 ? t.x : t.y;
  return eval_side(t, side, maps, s.nops, row, int(col - t.col0));
}
#endif

}  // namespace ttsw
