// Host-side tree / node layout (reference grid.py:204-322), native.
//
// Same closed forms as paper_1307_2665_b200/grid.py (TreeLayout._build), bit-exact with the
// reference's build_tree: heap-ordered boxes, one contiguous interior-id range per parent, uniform
// split maps per depth, and Gauss-node coordinates evaluated with the reference's fp64 expression
// order (compiled with -ffp-contract=off: no fused multiply-adds). The caller (grid.py) allocates
// every output; sizes follow from (L, q) alone. Every parent's split maps are checked, not a sample.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

struct Tree {
  int L, q;
  long long n;
  std::vector<long long> n3s, depth_off;

  // box footprint in leaf cells at depth d (cuts alternate vertical, horizontal)
  void shape(int d, long long& nx, long long& ny) const {
    nx = n >> ((d + 1) / 2);
    ny = n >> (d / 2);
  }
  // heap slot at depth d from box coordinates in units of that depth's box size (x bit first)
  static long long slot_from_xy(long long bx, long long by, int d) {
    long long slot = 0;
    const int nxb = (d + 1) / 2, nyb = d / 2;
    for (int t = 0; t < d; ++t) {
      const long long bit = (t % 2 == 0) ? (bx >> (nxb - 1 - t / 2)) & 1 : (by >> (nyb - 1 - t / 2)) & 1;
      slot = (slot << 1) | bit;
    }
    return slot;
  }
  static long long lowbit(long long v) { return v & -v; }
  static int log2i(long long v) {
    int r = 0;
    while ((1LL << r) < v) ++r;
    return r;
  }
  // id of the first Gauss node of segment `seg` on horizontal line `line` (key ('h', line, seg, 0))
  long long h_id(long long line, long long seg) const {
    if (line == 0) return seg * q;
    if (line == n) return 2 * n * q + seg * q;
    const long long low = lowbit(line), ny = 2 * low, nx = ny / 2;
    const int d = 2 * log2i(n / ny) + 1;
    const long long bx = seg / nx, by = (line - low) / ny;
    return depth_off[d] + slot_from_xy(bx, by, d) * n3s[d] + (seg - bx * nx) * q;
  }
  // the same on vertical line `line` (key ('v', line, seg, 0))
  long long v_id(long long line, long long seg) const {
    if (line == 0) return 3 * n * q + seg * q;
    if (line == n) return n * q + seg * q;
    const long long low = lowbit(line), nx = 2 * low, ny = nx;
    const int d = 2 * log2i(n / nx);
    const long long bx = (line - low) / nx, by = seg / ny;
    return depth_off[d] + slot_from_xy(bx, by, d) * n3s[d] + (seg - by * ny) * q;
  }
  void cells(int d, long long k, long long& ix, long long& iy) const {
    ix = iy = 0;
    for (int t = 0; t < d; ++t) {
      const long long bit = (k >> (d - 1 - t)) & 1;
      long long nx, ny;
      shape(t, nx, ny);
      if (t % 2 == 0)
        ix += bit * (nx / 2);
      else
        iy += bit * (ny / 2);
    }
  }
};

// body(lo, hi) over [0, n) split across up to 16 host threads (the big loops of a deep tree touch
// hundreds of MB for the first time; the page faults dominate and spread across cores)
template <class F>
void parallel_for(long long n, F body) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const long long nt = std::min<long long>(hw, std::max<long long>(1, n / 4096));
  if (nt <= 1) {
    body(0LL, n);
    return;
  }
  std::vector<std::thread> pool;
  const long long chunk = (n + nt - 1) / nt;
  for (long long t = 0; t < nt; ++t) {
    const long long lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) pool.emplace_back([=] { body(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

// Sizes of the layout of a 4^L-leaf tree with q Gauss nodes per leaf edge. n3[d], ne[d], m[d] for
// d < 2L (arrays of length max(2L, 1)); returns N (all Gauss nodes), or -1 on bad arguments.
extern "C" long long hps_tree_sizes(int L, int q, long long* n3, long long* ne, long long* m) {
  if (L < 0 || L > 20 || q < 1) {
    hps::set_error("hps_tree_sizes: bad L=%d q=%d", L, q);
    return -1;
  }
  const long long n = 1LL << L;
  long long N = 4 * n * q;
  for (int d = 0; d < 2 * L; ++d) {
    const long long nx = n >> ((d + 1) / 2), ny = n >> (d / 2);
    const long long n3d = (d % 2 == 0 ? ny : nx) * q;
    if (n3) n3[d] = n3d;
    if (ne) ne[d] = 2 * (nx + ny) * q;
    if (m) m[d] = (nx + ny) * q + n3d;  // |I_e(child)| = ne / 2 + n3
    N += (1LL << d) * n3d;
  }
  return N;
}

// The full layout. Inputs: L, q, the domain corner and extent, gauss01[q] = (gauss + 1) / 2 as the
// reference evaluates it. Outputs (caller-allocated): points[N][2], on_vertical[N],
// leaf_cells[4^L][2], leaf_I_e[4^L][4q], and per depth d < 2L: Ie[d] ([2^d][ne]), maps[d]
// (j1a[ne/2], j2b[ne/2], j3a[n3], j3b[n3]). Returns HPS_OK, or HPS_ERR_ARG if a parent's children
// do not share exactly its interior range or a depth's split maps are not uniform.
extern "C" int hps_tree_layout(int L, int q, double x_lo, double y_lo, double width, double height,
                               const double* gauss01, double* points, unsigned char* on_vertical,
                               long long* leaf_cells, long long* leaf_I_e, long long* const* Ie,
                               long long* const* maps) {
  Tree t;
  t.L = L;
  t.q = q;
  t.n = 1LL << L;
  const long long n = t.n;
  std::vector<long long> ne(2 * L + 1), mm(2 * L + 1);
  t.n3s.assign(2 * L + 1, 0);
  if (hps_tree_sizes(L, q, t.n3s.data(), ne.data(), mm.data()) < 0) return HPS_ERR_ARG;
  t.depth_off.assign(2 * L + 1, 0);
  t.depth_off[0] = 4 * n * q;
  for (int d = 0; d < 2 * L; ++d) t.depth_off[d + 1] = t.depth_off[d] + (1LL << d) * t.n3s[d];

  // coordinates (grid.py's expression order): line positions, Gauss offsets within a cell
  std::vector<double> xline(n + 1), yline(n + 1), gx(q), gy(q);
  const double hx = width / (double)n, hy = height / (double)n;
  for (long long i = 0; i <= n; ++i) {
    xline[i] = x_lo + (double)i * hx;
    yline[i] = y_lo + (double)i * hy;
  }
  for (int k = 0; k < q; ++k) {
    gx[k] = (x_lo + gauss01[k] * hx) - x_lo;
    gy[k] = gauss01[k] * hy;
  }
  auto put = [&](long long id, double x, double y, bool v) {
    points[2 * id] = x;
    points[2 * id + 1] = y;
    on_vertical[id] = v ? 1 : 0;
  };
  const long long nq = n * q;
  for (long long s = 0; s < n; ++s)
    for (int k = 0; k < q; ++k) {
      put(s * q + k, xline[s] + gx[k], yline[0], false);           // S
      put(nq + s * q + k, xline[n], yline[s] + gy[k], true);       // E
      put(2 * nq + s * q + k, xline[s] + gx[k], yline[n], false);  // N
      put(3 * nq + s * q + k, xline[0], yline[s] + gy[k], true);   // W
    }
  for (int d = 0; d < 2 * L; ++d) {
    long long nx, ny;
    t.shape(d, nx, ny);
    const long long n3 = t.n3s[d], nseg = n3 / q;
    parallel_for(1LL << d, [&, d, nx, ny, n3, nseg](long long k0, long long k1) {
      for (long long k = k0; k < k1; ++k) {
        long long ix, iy;
        t.cells(d, k, ix, iy);
        long long id = t.depth_off[d] + k * n3;
        for (long long sg = 0; sg < nseg; ++sg)
          for (int g = 0; g < q; ++g, ++id) {
            if (d % 2 == 0)  // vertical cut line x = ix + nx / 2, segments along y
              put(id, xline[ix + nx / 2], yline[iy + sg] + gy[g], true);
            else
              put(id, xline[ix + sg] + gx[g], yline[iy + ny / 2], false);
          }
      }
    });
  }

  // leaf boundary lists: S, E, N, W sides, increasing coordinate (grid.py:305-312)
  const long long nleaf = 1LL << (2 * L), m4 = 4LL * q;
  parallel_for(nleaf, [&](long long k0, long long k1) {
    for (long long k = k0; k < k1; ++k) {
      long long ix, iy;
      t.cells(2 * L, k, ix, iy);
      leaf_cells[2 * k] = ix;
      leaf_cells[2 * k + 1] = iy;
      long long* out = leaf_I_e + k * m4;
      const long long s0 = t.h_id(iy, ix), e0 = t.v_id(ix + 1, iy), n0 = t.h_id(iy + 1, ix), w0 = t.v_id(ix, iy);
      for (int g = 0; g < q; ++g) {
        out[g] = s0 + g;
        out[q + g] = e0 + g;
        out[2 * q + g] = n0 + g;
        out[3 * q + g] = w0 + g;
      }
    }
  });

  // parents bottom-up: child-a remainder then child-b remainder (grid.py:313-319)
  const long long* child = leaf_I_e;
  long long mchild = m4;
  for (int d = 2 * L - 1; d >= 0; --d) {
    const long long nb = 1LL << d, n3 = t.n3s[d], ned = ne[d], n1 = ned / 2;
    if (mchild != mm[d]) {
      hps::set_error("hps_tree_layout: child boundary length %lld != %lld at depth %d", mchild, mm[d], d);
      return HPS_ERR_ARG;
    }
    long long* j1a = maps[d];
    long long* j2b = j1a + n1;
    long long* j3a = j2b + n1;
    long long* j3b = j3a + n3;
    // maps from the first parent
    {
      const long long* A = child;
      const long long* B = child + mchild;
      const long long s0 = t.depth_off[d];
      long long c1 = 0, c2 = 0, c3a = 0, c3b = 0;
      for (long long p = 0; p < mchild; ++p) {
        if (A[p] >= s0 && A[p] < s0 + n3) {
          j3a[A[p] - s0] = p;
          ++c3a;
        } else if (c1 < n1) {
          j1a[c1++] = p;
        } else {
          c1 = n1 + 1;
        }
        if (B[p] >= s0 && B[p] < s0 + n3) {
          j3b[B[p] - s0] = p;
          ++c3b;
        } else if (c2 < n1) {
          j2b[c2++] = p;
        } else {
          c2 = n1 + 1;
        }
      }
      if (c3a != n3 || c3b != n3 || c1 != n1 || c2 != n1) {
        hps::set_error("hps_tree_layout: children are not edge-adjacent at depth %d", d);
        return HPS_ERR_ARG;
      }
    }
    long long* Id = Ie[d];
    std::vector<char> badflag(std::max<long long>(1, nb), 0);
    parallel_for(nb, [&](long long k0, long long k1) {
      for (long long k = k0; k < k1; ++k) {
        const long long* A = child + (2 * k) * mchild;
        const long long* B = child + (2 * k + 1) * mchild;
        const long long s0 = t.depth_off[d] + k * n3;
        for (long long i = 0; i < n3; ++i)  // every parent: the shared nodes are its I_i range
          if (A[j3a[i]] != s0 + i || B[j3b[i]] != s0 + i) badflag[k] = 1;
        long long* out = Id + k * ned;
        for (long long i = 0; i < n1; ++i) out[i] = A[j1a[i]];
        for (long long i = 0; i < n1; ++i) out[n1 + i] = B[j2b[i]];
      }
    });
    for (long long k = 0; k < nb; ++k)
      if (badflag[k]) {
        hps::set_error("hps_tree_layout: non-uniform split maps at depth %d (parent %lld)", d, k);
        return HPS_ERR_ARG;
      }
    child = Id;
    mchild = ned;
  }
  return HPS_OK;
}
