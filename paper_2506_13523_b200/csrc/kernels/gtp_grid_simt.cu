// Gaunt tensor products on the separable algorithm (large-L path), SIMT.
//
// Same algorithm as the reference (proj/src/sphere.cpp:105-195): Legendre
// synthesis per m, phi synthesis, pointwise product, phi analysis with the
// quadrature weights folded in, Legendre analysis.  O(L^3) per product
// instead of the dense GEMM formulation's O(L^4).
//   grid_quad_kernel  (below): four products per block as float4, both grid symmetries folded,
//                     register-tiled stages; the automatic path for the grid GTP and, on the
//                     reference torus folded to theta in [0, pi] (Context::fourier_sep), the
//                     Fourier GTP from L = 11
//   grid_simt_kernel  (first): one product per block, kept for comparison (TPO_GRID_SIMT_OLD) and
//                     for shapes whose row-quad shared memory does not fit
// All intermediates live in shared memory; blocks are persistent over rows.
// Also here: per-degree scaling, the backward's partial-sum accumulation and column gathers.
#include <algorithm>
#include <cstdlib>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    grid_simt_kernel(const __grid_constant__ GridSimtTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float sm[];
  const int nt = t.nt, np = t.np, B = t.band;
  const int din1 = (t.L1 + 1) * (t.L1 + 1), din2 = (t.L2 + 1) * (t.L2 + 1);
  const int nm1 = 2 * t.L1 + 1, nm2 = 2 * t.L2 + 1, nm3 = 2 * t.L3e + 1;
  float* xs = sm;                 // din1
  float* ys = xs + din1;          // din2
  float* gx = ys + din2;          // [nm1][nt]
  float* gy = gx + nm1 * nt;      // [nm2][nt]
  float* P = gy + nm2 * nt;       // [nt][np]
  float* h = P + nt * np;         // [nm3][nt]
  auto lam = [&](int l, int ma, int j) { return __ldg(t.lam + (l * (l + 1) / 2 + ma) * nt + j); };
  auto cs = [&](int m, int k) { return __ldg(t.cs + (m + B) * np + k); };
  for (int64_t row = blockIdx.x; row < rs.rows; row += gridDim.x) {
    const int64_t yr = rs.y_shared ? row / rs.channels : row;
    for (int i = threadIdx.x; i < din1; i += kThreads) xs[i] = __ldg(rs.x + row * din1 + i);
    for (int i = threadIdx.x; i < din2; i += kThreads) ys[i] = __ldg(rs.y + yr * din2 + i);
    __syncthreads();
    // 1. Legendre synthesis g_m(theta_j) = sum_{l>=|m|} x_lm Lambda_l|m|(theta_j)
    for (int i = threadIdx.x; i < (nm1 + nm2) * nt; i += kThreads) {
      const bool isx = i < nm1 * nt;
      const int ii = isx ? i : i - nm1 * nt;
      const int Lx = isx ? t.L1 : t.L2;
      const float* v = isx ? xs : ys;
      const int mi = ii / nt, j = ii - mi * nt, m = mi - Lx, ma = abs(m);
      float acc = 0.f;
      for (int l = ma; l <= Lx; ++l) acc = fmaf(v[l * l + m + l], lam(l, ma, j), acc);
      (isx ? gx : gy)[ii] = acc;
    }
    __syncthreads();
    // 2+3. phi synthesis of both inputs and pointwise product
    for (int i = threadIdx.x; i < nt * np; i += kThreads) {
      const int j = i / np, k = i - j * np;
      float fx = 0.f, fy = 0.f;
      for (int mi = 0; mi < nm1; ++mi) fx = fmaf(gx[mi * nt + j], cs(mi - t.L1, k), fx);
      for (int mi = 0; mi < nm2; ++mi) fy = fmaf(gy[mi * nt + j], cs(mi - t.L2, k), fy);
      P[i] = fx * fy;
    }
    __syncthreads();
    // 4. phi analysis, quadrature weight w_j * 2pi/n_phi folded in
    for (int i = threadIdx.x; i < nm3 * nt; i += kThreads) {
      const int mi = i / nt, j = i - mi * nt, m = mi - t.L3e;
      float acc = 0.f;
      for (int k = 0; k < np; ++k) acc = fmaf(P[j * np + k], cs(m, k), acc);
      h[i] = acc * __ldg(t.wq + j);
    }
    __syncthreads();
    // 5. Legendre analysis; degrees past the band are exactly zero
    for (int o = threadIdx.x; o < t.dout_total; o += kThreads) {
      float acc = 0.f;
      const int l = static_cast<int>(sqrtf(static_cast<float>(o)));
      const int lc = (l + 1) * (l + 1) <= o ? l + 1 : (l * l > o ? l - 1 : l);
      if (lc <= t.L3e) {
        const int m = o - lc * lc - lc, ma = abs(m);
        for (int j = 0; j < nt; ++j) acc = fmaf(h[(m + t.L3e) * nt + j], lam(lc, ma, j), acc);
      }
      rs.out[row * t.dout_total + o] = acc;
    }
    __syncthreads();
  }
}

}  // namespace

// ---------------------------------------------------------------- row-quad kernel
// The same five stages on a block of four products held as float4 (one lane of the vector per
// product), so every table coefficient and every staged value feeds four products, with both
// grid symmetries folded in:
//   phi:   phi_{np-k} = 2 pi - phi_k, so cos(m phi) is even and sin(m phi) odd about k = 0; the
//          synthesis evaluates E = sum_{m>=0} g_m cos and O = sum_{m<0} g_m sin on the half period
//          kp = 0..band and gives F(kp) = E + O, F(np - kp) = E - O; the analysis takes
//          S = P(kp) + P(np - kp) against cos and D = P(kp) - P(np - kp) against sin.
//   theta: the Gauss-Legendre nodes are symmetric, Lambda_lm(pi - theta) = (-1)^(l+m) Lambda_lm(theta),
//          so the Legendre synthesis sums even and odd l + m apart and the analysis reads
//          h(j) + h(j') or h(j) - h(j') by the parity of l + m.
// Each stage is a register-tiled small GEMM: stage 2 computes 4 half-period points x 4 products per
// thread for both inputs (32 FMAs per 3 loads), stage 4 a node pair x 4 orders x 4 products, stage 5
// two degrees of one order.  About half the FMAs of grid_simt_kernel and a fraction of its loads.
namespace {

constexpr int kQMaxThreads = 320;  // block = the larger of the stage-2 / stage-4 item counts, <= 320

// four products' FMAs as two packed f32x2 FMAs (FFMA2): half the FMA issue slots
__device__ __forceinline__ float4 f4fma(float4 a, float b, float4 c) {
  const float2 bb = make_float2(b, b);
  const float2 lo = __ffma2_rn(make_float2(a.x, a.y), bb, make_float2(c.x, c.y));
  const float2 hi = __ffma2_rn(make_float2(a.z, a.w), bb, make_float2(c.z, c.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ float4 f4mul(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
__device__ __forceinline__ float4 f4scale(float4 a, float b) { return make_float4(a.x * b, a.y * b, a.z * b, a.w * b); }
__device__ __forceinline__ float f4get(float4 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

struct QuadLayout {
  int din1, din2, nm1, nm2, nm3, nt, njp, nkp, dout_e;
  int regA, regB;  // float4 counts of the two aliased regions
  int trig;        // float4 count of the staged phi tables (c2c, c2s, c4c, c4s)
  int hoff;        // float4 offset of the h(j) - h(j') half of H: = 4 (mod 8), so that rows of the two
                   // halves land in different bank groups (rows step by njp, odd-ish strides collided)
};

__host__ __device__ inline QuadLayout quad_layout(const GridSimtTables& t) {
  QuadLayout q;
  q.din1 = (t.L1 + 1) * (t.L1 + 1);
  q.din2 = (t.L2 + 1) * (t.L2 + 1);
  q.nm1 = 2 * t.L1 + 1;
  q.nm2 = 2 * t.L2 + 1;
  q.nm3 = 2 * t.L3e + 1;
  q.nt = t.nt;
  q.njp = (t.nt + 1) / 2;
  q.nkp = t.nkp;
  q.dout_e = (t.L3e + 1) * (t.L3e + 1);
  q.hoff = q.nm3 * q.njp + ((4 - q.nm3 * q.njp % 8) + 8) % 8;
  const int a1 = (q.nm1 + q.nm2) * q.nt, a2 = q.hoff + q.nm3 * q.njp;
  const int b1 = q.din1 + q.din2, b2 = 2 * q.nt * q.nkp, b3 = q.dout_e;
  q.regA = a1 > a2 ? a1 : a2;
  q.regB = b1 > b2 ? (b1 > b3 ? b1 : b3) : (b2 > b3 ? b2 : b3);
  q.trig = ((t.band + 1) * t.nkpp * 2 + t.nkp * t.mpad * 2) / 4;
  return q;
}

template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    grid_quad_kernel(const __grid_constant__ GridSimtTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float4 sq[];
  const QuadLayout q = quad_layout(t);
  const int nt = q.nt, njp = q.njp, nkp = q.nkp, L1 = t.L1, L2 = t.L2, L3e = t.L3e;
  const int tid = threadIdx.x, nthr = blockDim.x;
  float4* A = sq;                // g = [nm1 + nm2][nt]         |  H = [2][nm3][njp] (h(j) +- h(j'))
  float4* B = sq + q.regA;       // xs, ys = [din1], [din2]  |  S, D = [nt][nkp]  |  outs (floats [4][dout_e])
  float4* gx = A;
  float4* gy = A + q.nm1 * nt;
  float4* H = A;
  float4* xs = B;
  float4* ys = B + q.din1;
  float4* S = B;
  float4* D = B + nt * nkp;
  float* outs = reinterpret_cast<float*>(B);
  // phi tables staged once per block (persistent over tiles): LDS instead of L1 round trips
  float4* trig = B + q.regB;
  const float4* c2c = trig;
  const float4* c2s = c2c + (t.band + 1) * t.nkpp / 4;
  const float4* c4c = c2s + (t.band + 1) * t.nkpp / 4;
  const float4* c4s = c4c + t.nkp * t.mpad / 4;
  {
    const int n2 = (t.band + 1) * t.nkpp / 4, n4 = t.nkp * t.mpad / 4;
    for (int i = tid; i < n2; i += nthr) {
      trig[i] = __ldg(reinterpret_cast<const float4*>(t.c2c) + i);
      trig[n2 + i] = __ldg(reinterpret_cast<const float4*>(t.c2s) + i);
    }
    for (int i = tid; i < n4; i += nthr) {
      trig[2 * n2 + i] = __ldg(reinterpret_cast<const float4*>(t.c4c) + i);
      trig[2 * n2 + n4 + i] = __ldg(reinterpret_cast<const float4*>(t.c4s) + i);
    }
  }
  const int64_t ntiles = (rs.rows + 3) / 4;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * 4;
    const int nr = static_cast<int>(rs.rows - row0 < 4 ? rs.rows - row0 : 4);
    // 0. stage the four products' inputs, product-minor: per coefficient the four rows' loads of
    //    both inputs in flight together, one float4 store each
    {
      const float* xr[4];
      const float* yr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t rr = row0 + (r < nr ? r : 0);
        xr[r] = rs.x + rr * q.din1;
        yr[r] = rs.y + (rs.y_shared ? rr / rs.channels : rr) * q.din2;
      }
      const int dmax = q.din1 > q.din2 ? q.din1 : q.din2;
      for (int k = tid; k < dmax; k += nthr) {
        float xv[4], yv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          xv[r] = (r < nr && k < q.din1) ? __ldg(xr[r] + k) : 0.f;
          yv[r] = (r < nr && k < q.din2) ? __ldg(yr[r] + k) : 0.f;
        }
        if (k < q.din1) xs[k] = make_float4(xv[0], xv[1], xv[2], xv[3]);
        if (k < q.din2) ys[k] = make_float4(yv[0], yv[1], yv[2], yv[3]);
      }
    }
    __syncthreads();
    // 1. Legendre synthesis on node pairs (j, nt-1-j), four first-half nodes per thread: even and odd
    //    l + |m| apart; running indices l^2 + l + m (input) and l (l + 1) / 2 + |m| (table row) step by
    //    2 l + 2 and l + 1
    {
      const int njq = t.njp4 / 4;
      for (int i = tid; i < (q.nm1 + q.nm2) * njq; i += nthr) {
        const int mi = i / njq, jq = i - mi * njq;
        const bool isx = mi < q.nm1;
        const int Lx = isx ? L1 : L2, m = (isx ? mi : mi - q.nm1) - Lx, ma = abs(m);
        const float4* v = isx ? xs : ys;
        float4 e[4], o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) e[c] = o[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        int vi = ma * ma + ma + m;
        const float4* lp = reinterpret_cast<const float4*>(t.lam1q + (ma * (ma + 1) / 2 + ma) * t.njp4) + jq;
        int l = ma;
        for (; l + 1 <= Lx; l += 2) {
          const float4 v0 = v[vi], w0 = __ldg(lp);
          vi += 2 * l + 2;
          lp += (l + 1) * njq;
          const float4 v1 = v[vi], w1 = __ldg(lp);
          vi += 2 * l + 4;
          lp += (l + 2) * njq;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            e[c] = f4fma(v0, f4get(w0, c), e[c]);
            o[c] = f4fma(v1, f4get(w1, c), o[c]);
          }
        }
        if (l <= Lx) {
          const float4 v0 = v[vi], w0 = __ldg(lp);
#pragma unroll
          for (int c = 0; c < 4; ++c) e[c] = f4fma(v0, f4get(w0, c), e[c]);
        }
        float4* g = (isx ? gx : gy) + (m + Lx) * nt;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int jp = jq * 4 + c;
          if (jp >= njp) break;
          g[jp] = f4add(e[c], o[c]);
          if (nt - 1 - jp != jp) g[nt - 1 - jp] = f4sub(e[c], o[c]);
        }
      }
    }
    __syncthreads();
    // 2+3. phi synthesis on the half period, product, folded into S / D.  m = 0 peeled (cos only),
    //      orders both inputs have in one branch-free loop, then each input's remaining orders
    {
      const int nkq = t.nkpp / 4, kq8 = nkq < 8 ? nkq : 8;
      const int Lc = L1 < L2 ? L1 : L2;
      for (int i = tid; i < nt * nkq; i += nthr) {
        // items (j, kq) in groups of <= 8 quads per node: a 128-bit shared load of 8 lanes then reads
        // 8 distinct table quads (9 quads per node put quads 0 and 8 in one bank group: 6-way conflicts)
        int j, kq;
        if (i < nt * kq8) {
          j = i / kq8;
          kq = i - j * kq8;
        } else {
          const int r2 = i - nt * kq8;
          kq = kq8 + r2 / nt;
          j = r2 - (kq - kq8) * nt;
        }
        float4 ex[4], ox[4], ey[4], oy[4];
        const float4* cp = c2c + kq;
        const float4* sp = c2s + kq;
        {
          const float4 cc = *cp;
          const float4 gxv = gx[L1 * nt + j], gyv = gy[L2 * nt + j];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ex[c] = f4scale(gxv, f4get(cc, c));
            ey[c] = f4scale(gyv, f4get(cc, c));
            ox[c] = oy[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        const float4* gxp = gx + (L1 + 1) * nt + j;  // order +m
        const float4* gxn = gx + (L1 - 1) * nt + j;  // order -m
        const float4* gyp = gy + (L2 + 1) * nt + j;
        const float4* gyn = gy + (L2 - 1) * nt + j;
        int m = 1;
        for (; m <= Lc; ++m) {
          cp += nkq;
          sp += nkq;
          const float4 cc = *cp, ss = *sp;
          const float4 a = *gxp, b = *gxn, c2 = *gyp, d = *gyn;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ex[c] = f4fma(a, f4get(cc, c), ex[c]);
            ox[c] = f4fma(b, f4get(ss, c), ox[c]);
            ey[c] = f4fma(c2, f4get(cc, c), ey[c]);
            oy[c] = f4fma(d, f4get(ss, c), oy[c]);
          }
          gxp += nt; gxn -= nt; gyp += nt; gyn -= nt;
        }
        for (int mx = m; mx <= L1; ++mx) {  // x orders past L2
          const float4 cc = cp[(mx - m + 1) * nkq], ss = sp[(mx - m + 1) * nkq];
          const float4 a = *gxp, b = *gxn;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ex[c] = f4fma(a, f4get(cc, c), ex[c]);
            ox[c] = f4fma(b, f4get(ss, c), ox[c]);
          }
          gxp += nt; gxn -= nt;
        }
        for (int my = m; my <= L2; ++my) {  // y orders past L1
          const float4 cc = cp[(my - m + 1) * nkq], ss = sp[(my - m + 1) * nkq];
          const float4 c2 = *gyp, d = *gyn;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ey[c] = f4fma(c2, f4get(cc, c), ey[c]);
            oy[c] = f4fma(d, f4get(ss, c), oy[c]);
          }
          gyp += nt; gyn -= nt;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int kp = kq * 4 + c;
          if (kp >= nkp) break;
          const float4 pp = f4mul(f4add(ex[c], ox[c]), f4add(ey[c], oy[c]));
          if (kp == 0) {
            S[j * nkp] = pp;
            D[j * nkp] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            const float4 pm = f4mul(f4sub(ex[c], ox[c]), f4sub(ey[c], oy[c]));
            S[j * nkp + kp] = f4add(pp, pm);
            D[j * nkp + kp] = f4sub(pp, pm);
          }
        }
      }
    }
    __syncthreads();
    // 4. phi analysis per node pair and order quad, quadrature weight folded in, stored as h(j) +- h(j')
    {
      const int nqc = (L3e + 1 + 3) / 4, nqs = (L3e + 3) / 4;
      for (int i = tid; i < njp * (nqc + nqs); i += nthr) {
        const bool sn = i >= njp * nqc;
        const int ii = sn ? i - njp * nqc : i;
        const int nq = sn ? nqs : nqc;
        const int nq8 = nq < 8 ? nq : 8;  // groups of <= 8 order quads per node pair (as stage 2)
        int jp, mq;
        if (ii < njp * nq8) {
          jp = ii / nq8;
          mq = ii - jp * nq8;
        } else {
          const int r2 = ii - njp * nq8;
          mq = nq8 + r2 / njp;
          jp = r2 - (mq - nq8) * njp;
        }
        const int j2 = nt - 1 - jp;
        const float4* src = sn ? D : S;
        const float4* tab = (sn ? c4s : c4c) + mq;
        const int mp4 = t.mpad / 4;
        float4 a0[4], a1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) a0[c] = a1[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int kp = sn ? 1 : 0; kp < nkp; ++kp) {
          const float4 cc = tab[kp * mp4];
          const float4 s0 = src[jp * nkp + kp], s1 = src[j2 * nkp + kp];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            a0[c] = f4fma(s0, f4get(cc, c), a0[c]);
            a1[c] = f4fma(s1, f4get(cc, c), a1[c]);
          }
        }
        const float w0 = __ldg(t.wq + jp), w1 = __ldg(t.wq + j2);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int mabs = sn ? mq * 4 + c + 1 : mq * 4 + c;
          if (mabs > L3e) break;
          const int mi = (sn ? -mabs : mabs) + L3e;
          const float4 h0 = f4scale(a0[c], w0);
          if (j2 == jp) {
            H[mi * njp + jp] = h0;
            H[q.hoff + mi * njp + jp] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            const float4 h1 = f4scale(a1[c], w1);
            H[mi * njp + jp] = f4add(h0, h1);
            H[q.hoff + mi * njp + jp] = f4sub(h0, h1);
          }
        }
      }
    }
    __syncthreads();
    // 5. Legendre analysis, two degrees of one order and parity per item
    for (int i = tid; i < t.nitems5; i += nthr) {
      const int it = __ldg(t.items5 + i);
      const int l0 = it & 0xffff, mi = it >> 16, m = mi - L3e, ma = abs(m);
      const int l1 = l0 + 2;
      const bool two = l1 <= L3e;
      const float4* h = H + ((l0 + ma) & 1) * q.hoff + mi * njp;
      const float2* w = reinterpret_cast<const float2*>(t.lam5t) + i;  // coalesced across the warp's items
      float4 c0 = make_float4(0.f, 0.f, 0.f, 0.f), c1 = c0;
#pragma unroll 4
      for (int jp = 0; jp < njp; ++jp) {
        const float4 hv = h[jp];
        const float2 wv = __ldg(w + jp * t.nitems5);
        c0 = f4fma(hv, wv.x, c0);
        c1 = f4fma(hv, wv.y, c1);
      }
      const int o0 = l0 * l0 + l0 + m;
      outs[0 * q.dout_e + o0] = c0.x;
      outs[1 * q.dout_e + o0] = c0.y;
      outs[2 * q.dout_e + o0] = c0.z;
      outs[3 * q.dout_e + o0] = c0.w;
      if (two) {
        const int o1 = l1 * l1 + l1 + m;
        outs[0 * q.dout_e + o1] = c1.x;
        outs[1 * q.dout_e + o1] = c1.y;
        outs[2 * q.dout_e + o1] = c1.z;
        outs[3 * q.dout_e + o1] = c1.w;
      }
    }
    __syncthreads();
    // 6. coalesced store; degrees past the band are exactly zero
#pragma unroll 1
    for (int r = 0; r < nr; ++r) {
      float* orow = rs.out + (row0 + r) * t.dout_total;
      const float* srow = outs + r * q.dout_e;
      for (int o = tid; o < t.dout_total; o += nthr) orow[o] = o < q.dout_e ? srow[o] : 0.f;
    }
    __syncthreads();
  }
}

size_t quad_smem(const GridSimtTables& t) {
  const QuadLayout q = quad_layout(t);
  return sizeof(float4) * static_cast<size_t>(q.regA + q.regB + q.trig);
}

// one pass over the two heavy stages' items where it fits: L = 16 has 297 / 289 items, which on 256
// threads took two passes (18.3 ms per 2^19 against 12.4 at L = 15 with 248 / 256 items)
int quad_threads(const GridSimtTables& t) {
  const QuadLayout q = quad_layout(t);
  const int i2 = q.nt * (t.nkpp / 4), i4 = q.njp * ((t.L3e + 4) / 4 + (t.L3e + 3) / 4);
  const int n = ((std::max(i2, i4) + 31) / 32) * 32;
  static const int forced = [] {  // sweeps only
    const char* v = std::getenv("TPO_QUAD_THREADS");
    return v ? std::atoi(v) : 0;
  }();
  if (forced > 0) return std::max(32, std::min(kQMaxThreads, forced / 32 * 32));
  return std::max(128, std::min(kQMaxThreads, n));
}

}  // namespace

bool gtp_grid_quad_fits(const GridSimtTables& t) { return quad_smem(t) <= 220 * 1024; }

cudaError_t launch_gtp_grid_simt(const GridSimtTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  static const bool old = std::getenv("TPO_GRID_SIMT_OLD") != nullptr;  // comparison only
  const size_t qsm = quad_smem(t);
  if ((!old || !t.lam) && qsm <= 220 * 1024) {
    const int nthr = quad_threads(t);
    static const int variant = [] {  // sweeps only: 256 / 320 forces that register budget
      const char* v = std::getenv("TPO_QUAD_VARIANT");
      return v ? std::atoi(v) : 0;
    }();
    // register budget by measurement (profiles/r02s/quad_variants2.jsonl): 90 registers (2 x 320
    // threads) at L <= 12 and 16, 110 (2 x 256) at 224 / 256 threads, i.e. L = 13..15 (-3..8%)
    const bool big = variant ? variant == 320 : (nthr > 256 || nthr < 224);
    // three 256-thread blocks per SM (80 registers) where their shared memory fits: L = 13 / 14
    // -2% / -4%; where it does not (L = 15) the register cap only costs (+7%)
    const bool three = !big && 3 * (qsm + 1024) <= 228 * 1024;
    auto kern = big ? grid_quad_kernel<320, 2> : (three ? grid_quad_kernel<256, 3> : grid_quad_kernel<256, 2>);
    if (nthr > 256 && !big) return cudaErrorInvalidValue;
    if (qsm > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(qsm));
      if (e != cudaSuccess) return e;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthr, qsm);
    const int64_t ntiles = (rs.rows + 3) / 4;
    const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
    kern<<<grid, nthr, qsm, s>>>(t, rs);
    return cudaGetLastError();
  }
  if (!t.lam) return cudaErrorInvalidValue;  // separable Fourier tables: row-quad kernel only
  const int din1 = (t.L1 + 1) * (t.L1 + 1), din2 = (t.L2 + 1) * (t.L2 + 1);
  const size_t smem = sizeof(float) * (din1 + din2 + (2 * t.L1 + 1 + 2 * t.L2 + 1) * t.nt + t.nt * t.np +
                                       (2 * t.L3e + 1) * t.nt);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(grid_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_simt_kernel, kThreads, smem);
  const int grid = static_cast<int>(std::min<int64_t>(rs.rows, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  grid_simt_kernel<<<grid, kThreads, smem, s>>>(t, rs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- per-degree scaling
namespace {
__global__ void scale_degrees_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n,
                                     int dim, int L, const float* __restrict__ w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(i % dim);
    int l = static_cast<int>(sqrtf(static_cast<float>(o)));
    if ((l + 1) * (l + 1) <= o) ++l;
    if (l * l > o) --l;
    out[i] = in[i] * __ldg(w + l);
  }
}
}  // namespace

cudaError_t launch_scale_degrees(const float* in, float* out, int64_t rows, int L, const float* w,
                                 cudaStream_t s) {
  const int dim = (L + 1) * (L + 1);
  const int64_t n = rows * dim;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  scale_degrees_kernel<<<grid, 256, 0, s>>>(in, out, n, dim, L, w);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- out += in (backward partial sums)
namespace {
__global__ void accumulate_kernel(const float4* __restrict__ in, float4* __restrict__ out, int64_t n4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(in + i);
    float4 b = out[i];
    b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
    out[i] = b;
  }
}
__global__ void accumulate_tail_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] += in[i];
}
}  // namespace

cudaError_t launch_accumulate(const float* in, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const bool vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const int64_t n4 = vec ? n / 4 : 0;
  if (n4 > 0) {
    const int grid = static_cast<int>(std::min<int64_t>((n4 + 255) / 256, 148 * 16));
    accumulate_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), n4);
  }
  const int64_t rem = n - 4 * n4;
  if (rem > 0)
    accumulate_tail_kernel<<<static_cast<int>((rem + 255) / 256), 256, 0, s>>>(in + 4 * n4, out + 4 * n4, rem);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- column window gather (backward)
namespace {
__global__ void gather_cols_kernel(const float* __restrict__ src, int64_t stride, int col0, int w,
                                   float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / w;
    dst[i] = __ldg(src + r * stride + col0 + (i - r * w));
  }
}
}  // namespace

cudaError_t launch_gather_cols(const float* src, int64_t stride, int col0, int w, float* dst, int64_t rows,
                               cudaStream_t s) {
  const int64_t n = rows * w;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  gather_cols_kernel<<<grid, 256, 0, s>>>(src, stride, col0, w, dst, n);
  return cudaGetLastError();
}

}  // namespace tpo_b200
