// Streaming matrix-free trace apply: warp-specialised, TMA-fed, persistent.
//
// Same operator as k_apply_local (CondensedSchur.apply_trace,
// condense.py:91-103; Algorithm 2 steps 1-4), restructured
// for the B200 memory system:
//   * sizes are compile-time (template <D, M, P>): every index is a constant
//     multiply/shift and every small loop unrolls;
//   * one producer warp streams each macro's operator data -- face blocks,
//     dG/dq stashes and the packed LU factor (packed_lu.cuh) -- in exactly
//     the order the math consumes it, as 1D bulk copies (cp.async.bulk, TMA)
//     into a ring of shared-memory stages guarded by mbarriers;
//   * eight consumer warps do all arithmetic out of shared memory, so the
//     bytes in flight are set by the ring depth, not by thread count;
//   * CTAs are persistent (grid = SMs x CTAs/SM) and walk the macros.
// Results match k_apply_local to rounding; all reductions are in a fixed order.
// Local trace entries are walked EPT = ceil(ltr / consumer threads) per thread (one for all
// configurations but 3D m = 2, p = 3, whose ltr = 560 exceeds the 512 consumer threads).
#include "dmma.cuh"
#include "local_ops.cuh"
#include "packed_lu.cuh"
#include "tiled_inv.cuh"
#include "tma.cuh"

namespace mhdg {

__host__ __device__ constexpr int cbinom(int n, int k) {
  int r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}
__host__ __device__ constexpr int cpow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
__host__ __device__ constexpr int ceven(int x) { return x + (x & 1); }

constexpr int ST_DBL = 2112;  // doubles per ring stage (16.5 KB: one 64x32 LU tile or a 64-row inverted triangle)
#ifndef MHDG_NCONS
#define MHDG_NCONS 512
#endif
#ifndef MHDG_STAGES
#define MHDG_STAGES 3
#endif
constexpr int NCONS = MHDG_NCONS;  // consumer threads of the pre / post / fused kernels (16 warps)

template <int D_, int M_, int P_>
struct Cfg {
  static constexpr int D = D_, M = M_, P = P_;
  static constexpr int NS = D + 2, NF = D + 1, N = M * P;
  static constexpr int L = cbinom(N + D, D), LF = cbinom(N + D - 1, D - 1);
  static constexpr int n = L * NS, BS = LF * NS, LTR = NF * BS;
  static constexpr int NSUB = cpow(M, D), NLOC = cbinom(P + D, D), NQ = cpow(P + 1, D);
  static constexpr int NTRI = cpow(M, D - 1), NLOCF = cbinom(P + D - 1, D - 1), NQF = cpow(P + 1, D - 1);
  static constexpr int NW = D * D * NS * NS, NWF = D * NS * NS;
  static constexpr int NPV = NSUB * NQ, NPF = NF * NTRI * NQF;
  // rows / points per ring stage (even counts where the unit has odd size)
  static constexpr int RPP = (BS & 1) ? ((ST_DBL / BS) & ~1) : ST_DBL / BS;
  static constexpr int PPV = (NW & 1) ? ((ST_DBL / NW) & ~1) : ST_DBL / NW;
  static constexpr int PPF = (NWF & 1) ? ((ST_DBL / NWF) & ~1) : ST_DBL / NWF;
  static constexpr int NBLK = (n + TI_RB - 1) / TI_RB;
  static constexpr int NFN = L - (N - 1 >= D ? cbinom(N - 1, D) : 0);  // boundary lattice nodes
};

enum : int { K_FST = 0, K_FTT, K_WV, K_WFZ, K_SI, K_Y2, K_FC, K_UNUSED, K_WF2, K_FTS, K_GF, K_MD };

struct Piece {
  unsigned char kind, blk;
  unsigned short u0, nu, cnt;  // cnt: doubles (even)
  unsigned off;                // doubles from the segment's per-macro (or table) base
};

__host__ __device__ constexpr int units_per_piece(int unit) {
  return (unit & 1) ? ((ST_DBL / unit) & ~1) < 1 ? 1 : ((ST_DBL / unit) & ~1) : (ST_DBL / unit) < 1 ? 1 : ST_DBL / unit;
}

// consumer-side ring cursor: stage index and phase in registers, barrier
// addresses precomputed
template <int STAGES>
struct ConsRing {
  uint32_t full0, empty0;
  const double* base;
  int stg = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ const double* wait() {
    mbar_wait_a(full0 + 8u * stg, ph);
    return base + stg * ST_DBL;
  }
  __device__ __forceinline__ void release(int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive_a(empty0 + 8u * stg);
    if (++stg == STAGES) {
      stg = 0;
      ph ^= 1u;
    }
  }
};

// consume the pieces of one segment: rows [u0, u0 + nu) of NROWS, PER per piece
template <int NROWS, int PER, class R, class Body>
__device__ __forceinline__ void seg_loop(R& rg, int lane, Body&& body) {
#pragma unroll 1
  for (int u0 = 0; u0 < NROWS; u0 += PER) {
    const double* A = rg.wait();
    body(A, u0, (NROWS - u0) < PER ? NROWS - u0 : PER);
    rg.release(lane);
  }
}

// Walks one macro's pieces in consumption order; the producer and the
// consumers run identical copies.  Segment order:
//   Gf table | FST | FTT | W_vol | W_face(z) | S^-1 tiles | y2, face terms | M^-1 D table | W_face(z2) | FTS
// PART 0 walks the fused apply (all but the hand-off pieces), PART 1 the
// segments before S^-1 (pre kernel), PART 2 the hand-off pieces and the
// segments after S^-1 (post kernel).
// MDR: the M^-1 D table stays resident in shared memory (post kernel) instead of streaming
// through the ring for every macro.
template <class C, int PART = 0, bool MDR = false>
struct Sched {
  int seg = 0, i = 0, b = 0, r = 0;
  // W_vol pieces hold whole sub-elements when they fit (one warp pass per point group)
  static constexpr bool WV_ALIGN = C::NQ * C::NW <= ST_DBL && ((C::NQ * C::NW) % 2 == 0);
  static constexpr int WV_PER = WV_ALIGN ? (ST_DBL / (C::NQ * C::NW)) * C::NQ : 0;
  __host__ __device__ bool rows(Piece& p, int kind, int nrows, int unit, int per = 0) {
    if (per <= 0) per = units_per_piece(unit);
    if (i * per >= nrows) return false;
    p.kind = (unsigned char)kind;
    p.u0 = (unsigned short)(i * per);
    p.nu = (unsigned short)(per < nrows - i * per ? per : nrows - i * per);
    p.off = (unsigned)((long long)p.u0 * unit);
    p.cnt = (unsigned short)ceven(p.nu * unit);
    p.blk = 0;
    ++i;
    return true;
  }
  __host__ __device__ bool next(Piece& p) {
    while (seg < 10) {
      if (PART == 1 && seg > 4) return false;  // pre part: up to the W_face(z) stash
      if (PART == 2 && seg < 6) {               // post part: from the hand-off pieces on
        seg = 6;
        i = r = b = 0;
      }
      switch (seg) {
        case 0: if (rows(p, K_GF, C::NF * C::L, C::LF)) return true; break;
        case 1: if (rows(p, K_FST, C::NF * C::BS, C::BS)) return true; break;
        case 2: if (rows(p, K_FTT, C::NF * C::BS, C::BS)) return true; break;
        case 3: if (rows(p, K_WV, C::NPV, C::NW, WV_PER)) return true; break;
        case 4: if (rows(p, K_WFZ, C::NPF, C::NWF)) return true; break;
        case 5:  // S^-1: row blocks of TI_RB rows, each as TI_CW-column tiles
          if (PART == 0 && b < C::NBLK) {
            const int nb = ti_rows(C::n, b);
            const int w = (C::n - r) < TI_CW ? C::n - r : TI_CW;
            p.kind = K_SI;
            p.u0 = (unsigned short)r;
            p.nu = (unsigned short)w;
            p.off = (unsigned)(ti_block_off(C::n, b) + (long long)(r / TI_CW) * nb * TI_CW);
            p.cnt = (unsigned short)ti_even((long long)nb * w);
            p.blk = (unsigned char)b;
            r += w;
            if (r >= C::n) { r = 0; ++b; }
            return true;
          }
          break;
        case 6:  // post part: y2 = S^-1 y1 and the pre part's face terms, from the work buffers
          if (PART == 2 && i < 2) {
            p.kind = (unsigned char)(i == 0 ? K_Y2 : K_FC);
            p.u0 = 0;
            p.nu = (unsigned short)(i == 0 ? C::n : C::LTR);
            p.off = 0;
            p.cnt = (unsigned short)(i == 0 ? ceven(C::n) : 2 * C::LTR);
            p.blk = 0;
            ++i;
            return true;
          }
          break;
        case 7: if (!MDR && rows(p, K_MD, C::D * C::NFN, C::L)) return true; break;
        case 8: if (rows(p, K_WF2, C::NPF, C::NWF)) return true; break;
        case 9: if (rows(p, K_FTS, C::NF * C::BS, C::BS)) return true; break;
      }
      ++seg;
      i = 0;
      r = 0;
      b = 0;
    }
    return false;
  }
};

// consumer work layout (doubles), after the ring; arrays a part does not use get
// no space (pre: x, z, y1, A_hh x, face terms, W results; post: y2, z2, A_hu y2, ...)
template <class C, int PART = 0>
struct SSm {
  static constexpr bool PRE = PART != 2, POST = PART != 1;
  static constexpr int xl = 0;
  static constexpr int z = xl + (PRE ? C::LTR : 0);  // z, later z2
  static constexpr int y = z + (PART == 2 ? C::D * C::NFN * C::NS : C::D * C::n);  // post: z2 at the face nodes only
  static constexpr int t = y + C::n;
  static constexpr int rfst = t + (PART == 0 ? C::n : 0);
  static constexpr int ftt = rfst + (PRE ? C::LTR : 0);
  static constexpr int fts = ftt + (PART == 2 ? 0 : C::LTR);  // post: A_hh x and g stay in registers
  static constexpr int cfgz = fts + (POST ? C::LTR : 0);
  static constexpr int yf = cfgz + (PART == 2 ? 0 : C::LTR);
  static constexpr int wfz = yf + (POST ? C::LTR : 0);
  static constexpr int wf2 = wfz + (PRE ? C::NPF * C::NS : 0);
  static constexpr int vv = wf2 + (POST ? C::NPF * C::NS : 0);  // one 32-double scratch per consumer warp
  static constexpr int cv = vv + (NCONS / 32) * 32;
  static constexpr int tg = cv + (PRE ? C::NSUB * C::NLOC * C::NS : 0);  // Gf x | W_vol results | M^-1 D y
  static constexpr int TGPRE = C::NF * C::n > C::NPV * C::D * C::NS ? C::NF * C::n : C::NPV * C::D * C::NS;
  static constexpr int TGPOST = C::D * C::NFN * C::NS;
  static constexpr int TGN = PART == 1 ? TGPRE : PART == 2 ? TGPOST : (TGPRE > TGPOST ? TGPRE : TGPOST);
  static constexpr int total = ceven(tg + TGN);
};

// Reference tables the consumers read, copied to shared memory once per CTA
// (after the work area): doubles first, then ints; the gradient classes
// (runtime count) go last.
template <class C>
struct TSm {
  static constexpr int phi_vol = 0;                             // NQ*NLOC
  static constexpr int phi_face = phi_vol + C::NQ * C::NLOC;    // NQF*NLOCF
  static constexpr int ndbl = ceven(phi_face + C::NQF * C::NLOCF);
  static constexpr int sub_conn = 0;                            // ints from here: NSUB*NLOC
  static constexpr int tri_conn = sub_conn + C::NSUB * C::NLOC;  // NTRI*NLOCF
  static constexpr int fvn = tri_conn + C::NTRI * C::NLOCF;      // NF*LF
  static constexpr int n2f = fvn + C::NF * C::LF;                // L
  static constexpr int fn_ptr = n2f + C::L;                      // LF+1
  static constexpr int fn_ent = fn_ptr + C::LF + 1;              // NTRI*NLOCF
  static constexpr int vf_ptr = fn_ent + C::NTRI * C::NLOCF;     // L+1
  static constexpr int vf_ent = vf_ptr + C::L + 1;               // NF*LF
  static constexpr int vn_ptr = vf_ent + C::NF * C::LF;          // L+1
  static constexpr int vn_sub = vn_ptr + C::L + 1;               // NSUB*NLOC
  static constexpr int gcls_of = vn_sub + C::NSUB * C::NLOC;     // NSUB
  static constexpr int nint = gcls_of + C::NSUB;
  static constexpr int total = ndbl + ceven((nint + 1) / 2);     // doubles
  static constexpr int CLS = C::NQ * C::NLOC * C::D;            // doubles per gradient class
};

// Post kernel with the macro-independent M^-1 D table (D NFN x L doubles: 52 KB at C2) resident
// in shared memory: streamed through the ring it was 52 of the 135 KB per macro the C2 post
// kernel moved.  Used when at least two ring stages still fit the two-CTAs-per-SM budget.
#ifndef MHDG_POST_MDR
#define MHDG_POST_MDR 1
#endif
template <class C>
__host__ __device__ constexpr int md_table() { return ceven(C::D * C::NFN * C::L); }
template <class C>
__host__ __device__ constexpr int post_stages_mdr() {
  return ((109 * 1024) / 8 - SSm<C, 2>::total - TSm<C>::total - md_table<C>()) / ST_DBL;
}
template <class C>
__host__ __device__ constexpr bool post_mdr() { return MHDG_POST_MDR != 0 && post_stages_mdr<C>() >= 2; }

__device__ __forceinline__ void cbar() { named_bar(1, NCONS); }

constexpr int NWARP_C = NCONS / 32;

// optional cycle accounting (build with -DMHDG_STREAM_PROFILE): per piece kind,
// [wait-for-data, compute, transition] cycles summed over CTAs (warp 0 lane 0)
#ifdef MHDG_STREAM_PROFILE
__device__ unsigned long long g_prof[16][3];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(k, j, v) atomicAdd(&g_prof[k][j], (unsigned long long)(clock64() - (v)))
#else
#define PROF_T(v)
#define PROF_ADD(k, j, v)
#endif
constexpr int MAXP = 256;  // pieces per macro (checked on the host)
// larger piece tables only for the configurations that need them (3D m = 2, p = 3: ~300 pieces);
// the others keep their static shared memory
template <class C>
__host__ __device__ constexpr int maxp_of() { return C::LTR > MHDG_NCONS ? 384 : MAXP; }

// First group >= g0 that warp `warp` owns when groups are dealt round-robin
// by global index over nw warps: consecutive pieces of one kind keep all warps busy.
__device__ __forceinline__ int first_group(int g0, int warp, int nw = NWARP_C) {
  return g0 + ((warp - g0 % nw) % nw + nw) % nw;
}

// The stash contractions (W_vol, W_face) hold ~10 quadrature points per ring stage:
// fewer point groups than consumer warps, and every group a dependent FMA chain.
// SPLIT consumption: the two halves of the consumer warps take alternate pieces, so
// two stages are contracted at once; every warp still waits for and releases every
// stage (the empty barrier counts all consumer warps), a warp skipping a piece only
// waits for it to land first.
constexpr int WSPLIT = 2;
template <int NROWS, int PER, class R, class Body>
__device__ __forceinline__ void seg_loop_split(R& rg, int lane, int warp, Body&& body) {
  constexpr int NWH = NWARP_C / WSPLIT;
  const int half = warp / NWH, wid = warp - half * NWH;
  int k = 0;
#pragma unroll 1
  for (int u0 = 0; u0 < NROWS; u0 += PER, ++k) {
    const double* A = rg.wait();
    if (k % WSPLIT == half) body(A, u0, (NROWS - u0) < PER ? NROWS - u0 : PER, wid, NWH);
    rg.release(lane);
  }
}

// acc_r = sum_c A[r][c] vec_r[c] for rows u0 .. u0+nu-1 of a staged piece, LPR
// lanes per row, RPW = 32/LPR rows per warp group, groups dealt to warps by
// global row index; out(r, acc) on one lane per row (r local to the piece).
template <int LPR, int NCOL, class VecF, class OutF>
__device__ __forceinline__ void rows_dot(const double* A, int u0, int nu, VecF vec, OutF out) {
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, l = lane % LPR;
  const int g1 = (u0 + nu - 1) / RPW;
  for (int gg = first_group(u0 / RPW, warp); gg <= g1; gg += NWARP_C) {
    const int rl = gg * RPW + sub - u0;
    const bool on = rl >= 0 && rl < nu;
    double a0 = 0.0, a1 = 0.0;
    if (on) {
      const double* a = A + rl * NCOL + l;
      const double* v = vec(rl) + l;
      constexpr int NK = (NCOL + LPR - 1) / LPR;  // columns l, l+LPR, ... (fixed trip count)
#pragma unroll
      for (int k = 0; k < NK; k += 2) {
        if (k * LPR + l < NCOL) a0 += a[k * LPR] * v[k * LPR];
        if (k + 1 < NK && (k + 1) * LPR + l < NCOL) a1 += a[(k + 1) * LPR] * v[(k + 1) * LPR];
      }
    }
    double acc = a0 + a1;
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(MHDG_FULL, acc, o);
    if (l == 0 && on) out(rl, acc);
  }
}

// Work buffers of the split apply (mhdg_factors.work), interleaved per macro so a
// contiguous macro range is a plain pointer offset (mhdg_apply_trace_local_range):
//   [M][ y1 (NP) | y2 (NP) | face terms: A_hh x (LTR) | g (LTR) ]   (NP = n rounded up to even)
template <class C>
struct Work {
  static constexpr int NP = ceven(C::n);
  static constexpr size_t PER = 2 * (size_t)NP + 2 * (size_t)C::LTR;
  static __host__ __device__ __forceinline__ double* y1(double* w, int m) { return w + (size_t)m * PER; }
  static __host__ __device__ __forceinline__ double* y2(double* w, int, int m) { return w + (size_t)m * PER + NP; }
  static __host__ __device__ __forceinline__ double* fc(double* w, int, int m) {
    return w + (size_t)m * PER + 2 * (size_t)NP;
  }
};

// Extra inputs that turn the pre part into the condensed rhs / recovery (condense.py:105-127):
// x == nullptr reads a zero trace; z += z_sign * z_add (the per-macro A_qq^-1 R_Q, layout
// (mac, l, node, s)); y1 += y1_sign * y1_add (R_U) before the hand-off.  All zero: the apply.
struct StreamIn {
  const double* z_add;
  double z_sign;
  const double* y1_add;
  double y1_sign;
};

template <class C, int STAGES, int PART>
__global__ void __launch_bounds__(NCONS + 32, (NCONS >= 1024 ? 1 : 2)) k_apply_stream(mhdg_disc g, mhdg_blocks bk, mhdg_factors fac,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ y_loc, int pref_ahead,
                                                             StreamIn sin) {
  constexpr int D = C::D, NS = C::NS, NF = C::NF, L = C::L, LF = C::LF, BS = C::BS, LTR = C::LTR, n = C::n;
  constexpr int NLOC = C::NLOC, NQ = C::NQ, NLOCF = C::NLOCF, NQF = C::NQF, NTRI = C::NTRI, NSUB = C::NSUB;
  // local trace entries per consumer thread (1 except where ltr > NCONS: 3D m = 2, p = 3);
  // entry e of thread tid is tid + j NCONS
  constexpr int EPT = (LTR + NCONS - 1) / NCONS;
  static_assert(2 * LTR <= ST_DBL, "the face-term hand-off piece must fit one ring stage");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ Piece pieces[maxp_of<C>()];
  __shared__ int npieces;
  __shared__ double cfls[16];  // z coefficients -(fac / det) area_f n_f,l of the current macro
  // z row of local node b of sub-face T of face f: [0] the volume node, [1] its face-node index
  __shared__ short fzn[2][C::NF * C::NTRI * C::NLOCF];
  using S = SSm<C, PART>;
  using TS = TSm<C>;
  constexpr bool MDRES = PART == 2 && post_mdr<C>();
  double* ring = smem;
  double* W = smem + STAGES * ST_DBL;
  double* Td = W + S::total;
  int* Ti = reinterpret_cast<int*>(Td + TS::ndbl);
  double* Gc = Td + TS::total;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long PK = ti_size(n);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NWARP_C);  // one arrival per consumer warp
    }
    fence_mbar_init();
    // the piece schedule is identical for every macro: build it once
    Sched<C, PART, MDRES> sc;
    int np = 0;
    while (np < maxp_of<C>() && sc.next(pieces[np])) ++np;
    npieces = np;
  }
  {  // reference tables -> shared memory
    const int nt = blockDim.x;
    for (int i = tid; i < NQ * NLOC; i += nt) Td[TS::phi_vol + i] = g.phi_vol[i];
    for (int i = tid; i < NQF * NLOCF; i += nt) Td[TS::phi_face + i] = g.phi_face[i];
    for (int i = tid; i < NSUB * NLOC; i += nt) {
      Ti[TS::sub_conn + i] = g.sub_conn[i];
      Ti[TS::vn_sub + i] = g.vn_sub[i];
    }
    for (int i = tid; i < NTRI * NLOCF; i += nt) {
      Ti[TS::tri_conn + i] = g.tri_conn[i];
      Ti[TS::fn_ent + i] = g.fn_ent[i];
    }
    for (int i = tid; i < NF * LF; i += nt) {
      Ti[TS::fvn + i] = g.face_vol_nodes[i];
      Ti[TS::vf_ent + i] = g.vf_ent[i];
    }
    for (int i = tid; i < L; i += nt) Ti[TS::n2f + i] = g.node_to_face[i];
    for (int i = tid; i <= L; i += nt) {
      Ti[TS::vf_ptr + i] = g.vf_ptr[i];
      Ti[TS::vn_ptr + i] = g.vn_ptr[i];
    }
    for (int i = tid; i <= LF; i += nt) Ti[TS::fn_ptr + i] = g.fn_ptr[i];
    for (int i = tid; i < NSUB; i += nt) Ti[TS::gcls_of + i] = g.grad_cls_of[i];
    for (int i = tid; i < NF * NTRI * NLOCF; i += nt) {
      const int f = i / (NTRI * NLOCF), tb = i % (NTRI * NLOCF);
      const int node = g.face_vol_nodes[f * LF + g.tri_conn[tb]];
      fzn[0][i] = (short)node;
      fzn[1][i] = (short)g.node_to_face[node];
    }
    if (PART != 2 && D == 2)  // 3D reads its (larger) class tables through L1
      for (int i = tid; i < g.n_grad_cls * TS::CLS; i += nt) Gc[i] = g.grad_cls[i];
    if (MDRES)  // the M^-1 D table, resident for the whole launch (the post part has no class tables)
      for (int i = tid; i < D * C::NFN * L; i += nt) Gc[i] = g.minv_d_face[i];
  }
  __syncthreads();
  const int np = npieces;

  // ----------------------------- producer ---------------------------------
  // One thread walks the (macro, piece) sequence: an optional prefetch cursor
  // pulls pieces from HBM into L2 pref_ahead pieces ahead, and the copy
  // cursor moves them into the shared ring once the consumers free a stage.
  if (warp == NWARP_C) {
    if (lane == 0) {
      auto src_of = [&](int mac, const Piece& p) -> const double* {
        switch (p.kind) {
          case K_GF: return g.gf + p.off;
          case K_MD: return g.minv_d_face + p.off;
          case K_FST: return bk.face_state_trace + (size_t)mac * NF * BS * BS + p.off;
          case K_FTT: return bk.face_trace_trace + (size_t)mac * NF * BS * BS + p.off;
          case K_FTS: return bk.face_trace_state + (size_t)mac * NF * BS * BS + p.off;
          case K_WV: return bk.wdgdq_vol + (size_t)mac * C::NPV * C::NW + p.off;
          case K_WFZ:
          case K_WF2: return bk.wdgdq_face + (size_t)mac * C::NPF * C::NWF + p.off;
          case K_Y2: return Work<C>::y2(fac.work, g.n_mac, mac);
          case K_FC: return Work<C>::fc(fac.work, g.n_mac, mac);
          default: return fac.lu + (size_t)mac * PK + p.off;  // S^-1 tiles
        }
      };
      // W_vol segments of an odd number of doubles (3D m = 1, p = 2: 27 x 225) leave every
      // other macro's base 8-byte aligned: those pieces are copied from one double earlier
      // (bulk copies need 16-byte alignment) and read from stage + 1
      constexpr bool WV_ODD = (C::NPV * C::NW) & 1;
      auto span = [&](int mac, const Piece& p, const double*& src, uint32_t& bytes) {
        src = src_of(mac, p);
        bytes = (uint32_t)p.cnt * 8u;
        if (WV_ODD && p.kind == K_WV && (mac & 1)) {
          src -= 1;
          bytes = (uint32_t)ceven(p.nu * C::NW + 1) * 8u;
        }
      };
      int pm = blockIdx.x, pp = 0, pref = 0;  // prefetch cursor (macro, piece), pieces issued
      int it = 0;
      for (int mac = blockIdx.x; mac < g.n_mac; mac += gridDim.x) {
        for (int pi = 0; pi < np; ++pi) {
          const Piece& p = pieces[pi];
          const int s = it % STAGES;
          while (pref < it + pref_ahead && pm < g.n_mac) {
            const Piece& q = pieces[pp];
            if (q.kind != K_GF && q.kind != K_MD && q.cnt) {
              const double* src;
              uint32_t nbytes;
              span(pm, q, src, nbytes);
              bulk_prefetch_l2(src, nbytes);
            }
            ++pref;
            if (++pp == np) { pp = 0; pm += gridDim.x; }
          }
          if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) + 1) & 1);
          const double* src;
          uint32_t bytes;
          span(mac, p, src, bytes);
          mbar_arrive_expect_tx(&full_bar[s], bytes);
          if (bytes) bulk_g2s(ring + s * ST_DBL, src, bytes, &full_bar[s]);
          ++it;
        }
      }
    }
    return;
  }

  // ----------------------------- consumers --------------------------------
  // The piece sequence is compile-time: each segment is a loop over its
  // pieces (ConsRing carries stage and phase), consumed in the order the
  // producer issues them (Sched).  Barriers only where data flows between
  // warps.
  double *xl = W + S::xl, *z = W + S::z, *y = W + S::y, *t = W + S::t, *rfst = W + S::rfst, *ftt = W + S::ftt,
         *fts = W + S::fts, *cfgz = W + S::cfgz, *yf = W + S::yf, *wfz = W + S::wfz, *wf2 = W + S::wf2,
         *vv = W + S::vv, *cv = W + S::cv, *tg = W + S::tg;
  const double *phs = Td + TS::phi_vol, *pfs = Td + TS::phi_face;
  const int *conn = Ti + TS::sub_conn, *tconn = Ti + TS::tri_conn, *fvn = Ti + TS::fvn, *n2f = Ti + TS::n2f,
            *fnp = Ti + TS::fn_ptr, *fne = Ti + TS::fn_ent, *vfp = Ti + TS::vf_ptr, *vfe = Ti + TS::vf_ent,
            *vnp = Ti + TS::vn_ptr, *vns = Ti + TS::vn_sub, *gco = Ti + TS::gcls_of;
  double* wv = tg;   // W_vol contraction results, lifetime: W_vol pieces .. y1
  double* z2 = z;    // z is dead once the W_face(z) pieces are consumed
  double* vw = vv + warp * 32;  // warp-private scratch
  using SC = Sched<C, PART, MDRES>;
  ConsRing<STAGES> rg{smem_u32(full_bar), smem_u32(empty_bar), ring};

  // this thread's trace entry of the next macro, gathered one macro ahead
  double x_next[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int e = tid + j * NCONS;
    x_next[j] = 0.0;
    if (PART != 2 && e < LTR && blockIdx.x < g.n_mac && x)
      x_next[j] = __ldg(x + __ldg(g.gather + (size_t)blockIdx.x * LTR + e));
  }

  auto zcoef = [&](int m) {  // -(fac / det) area_f n_f,l of macro m for this thread's (f, l)
    const int e = tid - (NCONS - NF * D), f = e / D;
    return -g.face_fac * __ldg(g.areas + m * NF + f) / __ldg(g.det + m) * __ldg(g.normals + (m * NF + f) * D + e % D);
  };
  double cfl_next = 0.0;
  if (PART != 2 && tid >= NCONS - NF * D && blockIdx.x < g.n_mac) cfl_next = zcoef(blockIdx.x);

  for (int mac = blockIdx.x; mac < g.n_mac; mac += gridDim.x) {
    double ij[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) ij[a][b] = __ldg(g.inv_jac + (size_t)mac * D * D + a * D + b);
    double sc_mine[EPT];  // trace_face_scale of this thread's face(s) in the final sum
    double ftt_mine[EPT], cfgz_mine[EPT];  // post part: this thread's A_hh x and g entries
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = tid + j * NCONS;
      sc_mine[j] = ftt_mine[j] = cfgz_mine[j] = 0.0;
      if (PART != 1 && e < LTR) sc_mine[j] = __ldg(bk.trace_face_scale + mac * NF + e / BS);
    }
    PROF_T(t_start);
    if (PART != 2 && tid >= NCONS - NF * D) {  // the last consumer threads: one z coefficient each,
      cfls[tid - (NCONS - NF * D)] = cfl_next;      // loaded one macro ahead like the trace entries
      const int nm = mac + gridDim.x;
      if (nm < g.n_mac) cfl_next = zcoef(nm);
    }
    if (PART != 2) {
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = tid + j * NCONS;
        if (e < LTR) {
          xl[e] = x_next[j];
          const int nm = mac + gridDim.x;
          if (nm < g.n_mac && x) x_next[j] = __ldg(x + __ldg(g.gather + (size_t)nm * LTR + e));
        }
      }
    }
    cbar();  // xl complete; the previous macro's readers of every work array are done
    if (tid == 0) { PROF_ADD(13, 2, t_start); }

    // W_vol / W_face contraction of one piece: v = phi z (gathered), out = W v.
    // Point groups of PPI points per warp pass, dealt to warps by global index.
    auto wcontract = [&](const double* A, int u0, int nu, bool face, bool second, int wid, int nw) {
      constexpr int DN = D * NS, PPI = 32 / DN;
      if constexpr (D == 3) {
        // 3D volume stash: 15 outputs of 15 terms per point and ~8 points per piece -- one point
        // per warp pass with two lanes per output (lane = 16 h + j; terms i = 2 i' + h, rotated by
        // 5 s: conflict-free W reads), so every warp of the half works on a piece and the
        // dependent FMA chains are half as long
        if (!face) {
          const int h = lane >> 4, j = lane & 15;
          const bool jon = j < DN;
          const int jj = jon ? j : 0, tt0 = jj % NS, l0 = jj / NS;  // v component / output (k, s)
          for (int pl = first_group(u0, wid, nw) - u0; pl < nu; pl += nw) {
            const int pt = u0 + pl, K = pt / NQ, q = pt % NQ;
            double a = 0.0;
#pragma unroll
            for (int b = 0; b < NLOC; b += 2)
              if (b + h < NLOC) a += phs[q * NLOC + b + h] * z[(l0 * L + conn[K * NLOC + b + h]) * NS + tt0];
            a += __shfl_xor_sync(MHDG_FULL, a, 16);
            if (h == 0 && jon) vw[j] = a;
            __syncwarp();
            const double* w = A + pl * C::NW + l0 * D * NS * NS + tt0 * NS;  // output k = l0, s = tt0
            double o = 0.0;
#pragma unroll
            for (int ip = 0; ip < (DN + 1) / 2; ++ip) {
              const int i = 2 * ip + h;
              if (i < DN) {
                int ii = i + NS * tt0;
                if (ii >= DN) ii -= DN;
                if (ii >= DN) ii -= DN;
                const int l = ii / NS, tt = ii - l * NS;
                o += w[l * NS * NS + tt] * vw[ii];
              }
            }
            o += __shfl_xor_sync(MHDG_FULL, o, 16);
            if (h == 0 && jon) wv[pt * DN + j] = o;
            __syncwarp();
          }
          return;
        }
      }
      const int pi = lane / DN, j = lane % DN;
      const int ngrp = (nu + PPI - 1) / PPI;
      for (int grp = first_group(u0 / PPI, wid, nw) - u0 / PPI; grp < ngrp; grp += nw) {
        const int pl = grp * PPI + pi;
        const bool on = pi < PPI && pl < nu;
        if (on) {
          const int tt = j % NS, l = j / NS;
          double a = 0.0;
          if (!face) {  // v[l][tt] = sum_b phi[q][b] z[l][conn[K][b]][tt]
            const int pt = u0 + pl, K = pt / NQ, q = pt % NQ;
#pragma unroll
            for (int b = 0; b < NLOC; ++b) a += phs[q * NLOC + b] * z[(l * L + conn[K * NLOC + b]) * NS + tt];
          } else {
            const double* zs = second ? z2 : z;
            const int lstride = second ? C::NFN : L;
            const int pf = u0 + pl, q = pf % NQF, T = (pf / NQF) % NTRI, f = pf / (NQF * NTRI);
#pragma unroll
            for (int b = 0; b < NLOCF; ++b) {
              const int node = fzn[second ? 1 : 0][(f * NTRI + T) * NLOCF + b];  // resolved once per CTA
              a += pfs[q * NLOCF + b] * zs[(l * lstride + node) * NS + tt];
            }
          }
          vw[pi * DN + j] = a;
        }
        __syncwarp();
        if (!face) {
          if (on) {  // out[k][s] = sum_{l,tt} W[k][l][s][tt] v[l][tt], (l, tt) order rotated per lane
            const int s = j % NS, k = j / NS;
            const double* w = A + pl * C::NW + k * D * NS * NS + s * NS;
            const double* v = vw + pi * DN;
            const int rot = (pi * D + k) % DN;
            double a = 0.0;
#pragma unroll
            for (int i = 0; i < DN; ++i) {
              int ii = i + rot;
              if (ii >= DN) ii -= DN;
              const int l = ii / NS, tt = ii - l * NS;
              a += w[l * NS * NS + tt] * v[ii];
            }
            wv[(u0 + pl) * DN + j] = a;
          }
        } else {
          // out[s] = sum_{l,tt} W[l][s][tt] v[l][tt]: lane (l, s) of the point's DN lanes sums over tt,
          // the D direction partials meet by shuffles (an NS-term chain instead of D NS)
          const int s = j % NS, l = j / NS;
          double a = 0.0;
          if (on) {
            const double* w = A + pl * C::NWF + l * NS * NS + s * NS;
            const double* v = vw + pi * DN + l * NS;
#pragma unroll
            for (int tt = 0; tt < NS; ++tt) a += w[tt] * v[tt];
          }
          double tot = a;
#pragma unroll
          for (int ll = 1; ll < D; ++ll) tot += __shfl_down_sync(MHDG_FULL, a, ll * NS);
          if (on && j < NS) (second ? wf2 : wfz)[(u0 + pl) * NS + s] = tot;
        }
        __syncwarp();
      }
    };

    // y1 = -A_uh x + A_uq z (needs rfst, the W_vol results, the W_face(z) stash);
    // leaves y1 in y and the face term g = A_hq z / scale in cfgz
    auto make_y1 = [&]() {
      // cv[K][a][s] = sum_q sum_k gphys[K,q,a,k] w[K,q][k][s], gphys = grad_ref[K] inv_jac
      if constexpr (D == 3) {
        // 3D: w'[q][r][s] = sum_k inv_jac[r][k] w[q][k][s] in place, then
        // cv = sum_{q,r} G_cls[q][a][r] w'[q][r][s] with the class tables read through L1
        constexpr int DN = D * NS;
        for (int idx = tid; idx < C::NPV * NS; idx += NCONS) {
          const int pt = idx / NS, s = idx - pt * NS;
          double w[D];
#pragma unroll
          for (int k = 0; k < D; ++k) w[k] = wv[pt * DN + k * NS + s];
#pragma unroll
          for (int r = 0; r < D; ++r) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) v += ij[r][k] * w[k];
            wv[pt * DN + r * NS + s] = v;
          }
        }
        cbar();
        for (int idx = tid; idx < NSUB * NLOC * NS; idx += NCONS) {
          const int s = idx % NS, a = (idx / NS) % NLOC, K = idx / (NS * NLOC);
          const double* G = g.grad_cls + (size_t)gco[K] * TS::CLS + a * D;
          const double* w = wv + K * NQ * DN + s;
          double ar[D] = {};  // one chain per direction r: D independent FMA chains
#pragma unroll 9
          for (int q = 0; q < NQ; ++q) {
#pragma unroll
            for (int r = 0; r < D; ++r) ar[r] += __ldg(G + q * NLOC * D + r) * w[(q * D + r) * NS];
          }
          double sum = ar[0];
#pragma unroll
          for (int r = 1; r < D; ++r) sum += ar[r];
          cv[idx] = sum;
        }
      } else {
        // 2D: per sub-element an (NLOC x NQ D) x (NQ D x NS) product on the FP64 tensor cores --
        // units (K, 8-row tile of a) dealt to the warps; the A fragments are gphys formed on the
        // fly from the class tables in shared memory and inv_jac, the B fragments the W_vol
        // results; two accumulator chains (even / odd k-steps).  (3D keeps the FFMA loop: its
        // class tables are read through L1 and 21 fragment loads in flight do not fit the
        // register budget -- measured pre 5.02 -> 5.32 ms.)
        constexpr int DN = D * NS, MT = (NLOC + 7) / 8, KD = NQ * D, KST = (KD + 3) / 4;
        const int g8 = lane >> 2, t4 = lane & 3;
        for (int un = warp; un < NSUB * MT; un += NWARP_C) {
          const int K = un / MT, a = (un - K * MT) * 8 + g8;
          const bool aok = a < NLOC;
          const double* G = Gc + gco[K] * TS::CLS + (aok ? a : 0) * D;
          const double* w = wv + K * NQ * DN + (g8 < NS ? g8 : 0);
          double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll 2
          for (int ks = 0; ks < KST; ks += 2) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int kk = 4 * (ks + hh) + t4;
              if (ks + hh < KST) {
                const bool kok = kk < KD;
                const int q = kok ? kk / D : 0, k = kok ? kk - q * D : 0;
                double af = 0.0;
#pragma unroll
                for (int r = 0; r < D; ++r) {
                  double ijk = ij[r][0];
#pragma unroll
                  for (int k2 = 1; k2 < D; ++k2) ijk = k == k2 ? ij[r][k2] : ijk;
                  af += G[q * NLOC * D + r] * ijk;
                }
                if (!(aok && kok)) af = 0.0;
                const double bf = (kok && g8 < NS) ? w[q * DN + k * NS] : 0.0;
                if (hh == 0) dmma_8x8x4(c0, c1, af, bf);
                else dmma_8x8x4(e0, e1, af, bf);
              }
            }
          }
          const int s0 = 2 * t4;
          if (aok && s0 < NS) cv[(K * NLOC + a) * NS + s0] = c0 + e0;
          if (aok && s0 + 1 < NS) cv[(K * NLOC + a) * NS + s0 + 1] = c1 + e1;
        }
      }
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int idx = tid + j * NCONS;
        if (idx < LTR) {
          const int s = idx % NS, gg = (idx / NS) % LF, f = idx / BS;
          double acc = 0.0;
          for (int e = fnp[gg]; e < fnp[gg + 1]; ++e) {
            const int ent = fne[e], T = ent / NLOCF, a = ent % NLOCF;
            const double* w = wfz + ((f * NTRI + T) * NQF) * NS + s;
#pragma unroll
            for (int q = 0; q < NQF; ++q) acc += pfs[q * NLOCF + a] * w[q * NS];
          }
          cfgz[idx] = acc;
        }
      }
      cbar();
      for (int idx = tid; idx < n; idx += NCONS) {
        const int I = idx / NS, s = idx % NS;
        double st = 0.0, sg = 0.0;
        for (int e = vfp[I]; e < vfp[I + 1]; ++e) st += rfst[vfe[e] * NS + s];
        for (int e = vnp[I]; e < vnp[I + 1]; ++e) sg -= cv[vns[e] * NS + s];
        for (int e = vfp[I]; e < vfp[I + 1]; ++e) sg += cfgz[vfe[e] * NS + s];
        y[idx] = -st + sg;
      }
      cbar();
    };

    if (PART != 2) {
      PROF_T(t0);
      // tg[f][I][s] = sum_h Gf[f][I][h] x[f][h][s]
      seg_loop<NF * L, units_per_piece(LF)>(rg, lane, [&](const double* A, int u0, int nu) {
        for (int idx = tid; idx < nu * NS; idx += NCONS) {
          const int s = idx % NS, rl = idx / NS, row = u0 + rl, f = row / L;
          const double* a = A + rl * LF;
          const double* xf = xl + f * BS + s;
          double acc = 0.0;
#pragma unroll
          for (int h = 0; h < LF; ++h) acc += a[h] * xf[h * NS];
          tg[row * NS + s] = acc;
        }
      });
      if (tid == 0) { PROF_ADD(K_GF, 1, t0); }
      PROF_T(t1);
      cbar();
      {  // z = A_qq^-1 A_qh x = -(fac/det) sum_f area_f n_f (Gf x_f); the coefficients were
         // put in shared memory at the start of the macro (their global loads ran under the Gf phase)
        double cfl[NF][D];
#pragma unroll
        for (int f = 0; f < NF; ++f)
#pragma unroll
          for (int l = 0; l < D; ++l) cfl[f][l] = cfls[f * D + l];
        for (int idx = tid; idx < n; idx += NCONS) {
          double acc[D] = {};
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const double tv = tg[f * n + idx];
#pragma unroll
            for (int l = 0; l < D; ++l) acc[l] += cfl[f][l] * tv;
          }
          if (PART == 1 && sin.z_add) {
            const double* za = sin.z_add + (size_t)mac * D * n + idx;
#pragma unroll
            for (int l = 0; l < D; ++l) z[l * n + idx] = acc[l] + sin.z_sign * __ldg(za + l * n);
          } else {
#pragma unroll
            for (int l = 0; l < D; ++l) z[l * n + idx] = acc[l];
          }
        }
      }
      cbar();  // z complete; tg free for the W_vol results
      if (tid == 0) { PROF_ADD(K_FST, 2, t1); }
      PROF_T(t2);
      seg_loop<NF * BS, units_per_piece(BS)>(rg, lane, [&](const double* A, int u0, int nu) {
        rows_dot<4, BS>(A, u0, nu, [&](int rl) { return xl + ((u0 + rl) / BS) * BS; },
                        [&](int rl, double acc) { rfst[u0 + rl] = acc; });
      });
      if (tid == 0) { PROF_ADD(K_FST, 1, t2); }
      PROF_T(t3);
      seg_loop<NF * BS, units_per_piece(BS)>(rg, lane, [&](const double* A, int u0, int nu) {
        rows_dot<4, BS>(A, u0, nu, [&](int rl) { return xl + ((u0 + rl) / BS) * BS; },
                        [&](int rl, double acc) { ftt[u0 + rl] = acc; });
      });
      if (tid == 0) { PROF_ADD(K_FTT, 1, t3); }
      PROF_T(t4);
      seg_loop_split<C::NPV, SC::WV_ALIGN ? SC::WV_PER : units_per_piece(C::NW)>(
          rg, lane, warp, [&](const double* A, int u0, int nu, int wid, int nw) {
            wcontract(A + (((C::NPV * C::NW) & 1) && (mac & 1) ? 1 : 0), u0, nu, false, false, wid, nw);
          });
      if (tid == 0) { PROF_ADD(K_WV, 1, t4); }
      PROF_T(t5);
      seg_loop_split<C::NPF, units_per_piece(C::NWF)>(
          rg, lane, warp, [&](const double* A, int u0, int nu, int wid, int nw) {
            wcontract(A, u0, nu, true, false, wid, nw);
          });
      if (tid == 0) { PROF_ADD(K_WFZ, 1, t5); }
      PROF_T(t6);
      cbar();  // rfst, W_vol results, W_face(z) stash complete
      make_y1();
      if (tid == 0) { PROF_ADD(14, 1, t6); }
    }
    if (PART == 1) {  // hand y1 and the face terms to the S^-1 stream / post kernels
      PROF_T(t_wb);
      double* y1g = Work<C>::y1(fac.work, mac);
      if (sin.y1_add) {
        const double* ya = sin.y1_add + (size_t)mac * n;
        for (int i = tid; i < n; i += NCONS) y1g[i] = y[i] + sin.y1_sign * __ldg(ya + i);
      } else {
        for (int i = tid; i < n; i += NCONS) y1g[i] = y[i];
      }
      double* fc = Work<C>::fc(fac.work, g.n_mac, mac);
      for (int e = tid; e < LTR; e += NCONS) {
        fc[e] = ftt[e];
        fc[LTR + e] = cfgz[e];
      }
      if (tid == 0) { PROF_ADD(15, 2, t_wb); }
      continue;  // the next macro's first barrier orders these reads before any overwrite
    }
    if (PART == 0) {  // y2 = S^-1 y1: row blocks of column tiles; warp w owns rows SRW*w.. of every block
      constexpr int SRW = TI_RB / NWARP_C, SLR = 32 / SRW;
      static_assert(SRW * NWARP_C == TI_RB && SRW * SLR == 32, "S^-1 tile mapping");
      PROF_T(t7);
      for (int b = 0; b < C::NBLK; ++b) {
        const int nb = ti_rows(n, b);
        const int r = SRW * warp + lane / SLR, l = lane % SLR;
        double acc = 0.0;
        for (int c0 = 0; c0 < n; c0 += TI_CW) {
          const int w = (n - c0) < TI_CW ? n - c0 : TI_CW;
          const double* A = rg.wait();
          if (r < nb) {
            const double* a = A + r * w;
            const double* yv = y + c0;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int k = 0; k < TI_CW / SLR; k += 2) {
              const int c = l + SLR * k;
              if (c < w) a0 += a[c] * yv[c];
              if (c + SLR < w) a1 += a[c + SLR] * yv[c + SLR];
            }
            acc += a0 + a1;
          }
          rg.release(lane);
        }
#pragma unroll
        for (int o = SLR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(MHDG_FULL, acc, o);
        if (l == 0 && r < nb) t[b * TI_RB + r] = acc;
      }
      cbar();
      for (int i = tid; i < n; i += NCONS) y[i] = t[i];
      if (tid == 0) { PROF_ADD(K_SI, 1, t7); }
    } else {  // post part: y2 and the pre part's face terms arrive as the first two pieces
      PROF_T(t8);
      seg_loop<1, 1>(rg, lane, [&](const double* A, int, int) {
        for (int i = tid; i < n; i += NCONS) y[i] = A[i];
      });
      seg_loop<1, 1>(rg, lane, [&](const double* A, int, int) {
#pragma unroll
        for (int j = 0; j < EPT; ++j) {  // this thread's entries, used by the same thread in the final sum
          const int e = tid + j * NCONS;
          if (e < LTR) {
            ftt_mine[j] = A[e];
            cfgz_mine[j] = A[LTR + e];
          }
        }
      });
      if (tid == 0) { PROF_ADD(K_Y2, 1, t8); }
    }
    PROF_T(t9);
    cbar();  // y = y2 complete
    for (int idx = tid; idx < LTR; idx += NCONS) {  // y2 restricted to the face nodes, for A_hu
      const int s = idx % NS, h = (idx / NS) % LF, f = idx / BS;
      yf[idx] = y[fvn[f * LF + h] * NS + s];
    }
    // tg[r][i][s] = sum_J (M^-1 D_r)[fnode_i][J] y2[J][s]: lane = (J half, row, s) for groups
    // of MDR rows dealt to warps by global index; the two halves meet in one shuffle
    // On the FP64 tensor cores: 8-row tiles of the table (A fragments straight from shared
    // memory) against y2 as an L x NS matrix padded to 8 columns; two accumulator chains (even
    // and odd k-steps), tiles dealt to warps by global index.
    auto md_rows = [&](const double* A, int u0, int nu) {
      const int g8 = lane >> 2, t4 = lane & 3;
      constexpr int KSTEPS = (L + 3) / 4;
      const int t1 = (u0 + nu - 1) / 8;
      for (int tt = first_group(u0 / 8, warp); tt <= t1; tt += NWARP_C) {
        const int row = tt * 8 + g8;
        const bool on = row >= u0 && row < u0 + nu;
        const double* a = A + (on ? row - u0 : 0) * L;
        double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll 4
        for (int ks = 0; ks < KSTEPS; ks += 2) {
          {
            const int J = 4 * ks + t4;
            const double af = (on && J < L) ? a[J] : 0.0;
            const double bf = (g8 < NS && J < L) ? y[J * NS + g8] : 0.0;
            dmma_8x8x4(c0, c1, af, bf);
          }
          if (ks + 1 < KSTEPS) {
            const int J = 4 * (ks + 1) + t4;
            const double af = (on && J < L) ? a[J] : 0.0;
            const double bf = (g8 < NS && J < L) ? y[J * NS + g8] : 0.0;
            dmma_8x8x4(e0, e1, af, bf);
          }
        }
        const int s0 = 2 * t4;
        if (on && s0 < NS) tg[row * NS + s0] = c0 + e0;
        if (on && s0 + 1 < NS) tg[row * NS + s0 + 1] = c1 + e1;
      }
    };
    if constexpr (MDRES) md_rows(Gc, 0, D * C::NFN);  // the resident table, all rows at once
    else seg_loop<D * C::NFN, units_per_piece(L)>(rg, lane, md_rows);
    if (tid == 0) { PROF_ADD(K_MD, 1, t9); }
    PROF_T(t10);
    cbar();
    {  // z2 = A_qq^-1 A_qu y2 = sum_r inv_jac[r][l] (M^-1 D_r y2), at the face nodes only
      constexpr int FNS = C::NFN * NS;
      for (int idx = tid; idx < FNS; idx += NCONS) {
        double tr[D];
#pragma unroll
        for (int r = 0; r < D; ++r) tr[r] = tg[r * FNS + idx];
#pragma unroll
        for (int l = 0; l < D; ++l) {
          double v = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) v += ij[r][l] * tr[r];
          z2[l * FNS + idx] = v;
        }
      }
    }
    cbar();  // z2 and yf complete
    if (tid == 0) { PROF_ADD(K_WF2, 2, t10); }
    PROF_T(t11);
    seg_loop_split<C::NPF, units_per_piece(C::NWF)>(
        rg, lane, warp, [&](const double* A, int u0, int nu, int wid, int nw) {
          wcontract(A, u0, nu, true, true, wid, nw);
        });
    seg_loop<NF * BS, units_per_piece(BS)>(rg, lane, [&](const double* A, int u0, int nu) {
      rows_dot<4, BS>(A, u0, nu, [&](int rl) { return yf + ((u0 + rl) / BS) * BS; },
                      [&](int rl, double acc) { fts[u0 + rl] = acc; });
    });
    if (tid == 0) { PROF_ADD(K_FTS, 1, t11); }
    PROF_T(t_end);
    cbar();  // wf2, fts complete

    // y4 = ((A_hu y2 - A_hq z2) + A_hh x) - A_hq z, with -A_hq z = scale * cfg
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int idx = tid + j * NCONS;
      if (idx < LTR) {
        const int s = idx % NS, gg = (idx / NS) % LF, f = idx / BS;
        double acc = 0.0;
        for (int e = fnp[gg]; e < fnp[gg + 1]; ++e) {
          const int ent = fne[e], T = ent / NLOCF, a = ent % NLOCF;
          const double* w = wf2 + ((f * NTRI + T) * NQF) * NS + s;
#pragma unroll
          for (int q = 0; q < NQF; ++q) acc += pfs[q * NLOCF + a] * w[q * NS];
        }
        y_loc[(size_t)mac * LTR + idx] = ((fts[idx] + sc_mine[j] * acc) + (PART == 2 ? ftt_mine[j] : ftt[idx])) +
                                         sc_mine[j] * (PART == 2 ? cfgz_mine[j] : cfgz[idx]);
      }
    }
    if (tid == 0) { PROF_ADD(12, 2, t_end); }
  }
}

// ---------------------------------------------------------------------------
// S^-1 stream (split apply, middle kernel): y2 = S^-1 y1 for every macro.
//
// Pure streaming batched GEMV over the tiled inverse (tiled_inv.cuh): 76% of
// the apply's bytes at C2 and no other work, so it runs with several CTAs per
// SM and a TMA ring each.  Work units are (macro, 64-row block) pairs, split
// contiguously across CTAs so consecutive units share the macro and y1 is
// fetched once per macro (as the first ring piece).  Consumer mapping: warp w
// owns rows SRW*w .. SRW*w+SRW-1 of the block, lane l column c0+l of every
// tile: the lanes of one row read 32 consecutive doubles (conflict-free) and
// each lane reads y once per tile; partial sums stay in registers across the
// block's tiles and are reduced across lanes once per unit.
// ---------------------------------------------------------------------------
template <class C, int STAGES, int NCT>
__global__ void __launch_bounds__(NCT + 32) k_si_stream(int n_mac, const double* __restrict__ inv,
                                                       double* __restrict__ work) {
  constexpr int n = C::n, NP = ceven(n), NBLK = C::NBLK, NT = (n + TI_CW - 1) / TI_CW;
  constexpr int NW = NCT / 32, SRW = TI_RB / NW;
  static_assert(SRW * NW == TI_RB && TI_CW == 32, "S^-1 stream mapping");
  static_assert(NP <= ST_DBL, "y1 must fit one ring stage");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  double* ring = smem;
  double* ybuf = smem + STAGES * ST_DBL;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long PK = ti_size(n);
  const long long U = (long long)n_mac * NBLK;
  const long long u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // producer: y1 of each new macro, then the block's column tiles
    if (lane == 0) {
      int it = 0, cur = -1;
      for (long long u = u0; u < u1; ++u) {
        const int mac = (int)(u / NBLK), b = (int)(u % NBLK), nb = ti_rows(n, b);
        const bool fresh = mac != cur;
        for (int k = fresh ? -1 : 0; k < NT; ++k) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) + 1) & 1);
          const double* src;
          uint32_t bytes;
          if (k < 0) {
            src = Work<C>::y1(work, mac);
            bytes = NP * 8u;
          } else {
            const int w = (n - k * TI_CW) < TI_CW ? n - k * TI_CW : TI_CW;
            src = inv + (size_t)mac * PK + ti_block_off(n, b) + (long long)k * nb * TI_CW;
            bytes = (uint32_t)ti_even((long long)nb * w) * 8u;
          }
          mbar_arrive_expect_tx(&full_bar[s], bytes);
          bulk_g2s(ring + s * ST_DBL, src, bytes, &full_bar[s]);
          ++it;
        }
        cur = mac;
      }
    }
    return;
  }

  int it = 0, cur = -1;
  for (long long u = u0; u < u1; ++u) {
    const int mac = (int)(u / NBLK), b = (int)(u % NBLK), nb = ti_rows(n, b);
    if (mac != cur) {
      named_bar(1, NCT);  // every warp is done with the previous macro's y1
      const int s = it % STAGES;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      for (int i = tid; i < NP; i += NCT) ybuf[i] = ring[s * ST_DBL + i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      ++it;
      named_bar(1, NCT);
      cur = mac;
    }
    double acc[SRW];
#pragma unroll
    for (int j = 0; j < SRW; ++j) acc[j] = 0.0;
    const int r0 = SRW * warp;
#pragma unroll 1
    for (int k = 0; k < NT; ++k) {
      const int s = it % STAGES;
      const int c0 = k * TI_CW, w = (n - c0) < TI_CW ? n - c0 : TI_CW;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      const double* A = ring + s * ST_DBL;
      if (lane < w) {
        const double yv = ybuf[c0 + lane];
#pragma unroll
        for (int j = 0; j < SRW; ++j)
          if (r0 + j < nb) acc[j] += A[(r0 + j) * w + lane] * yv;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      ++it;
    }
    double* y2 = Work<C>::y2(work, n_mac, mac) + b * TI_RB;
#pragma unroll
    for (int j = 0; j < SRW; ++j) {
      double v = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MHDG_FULL, v, o);
      if (lane == j && r0 + j < nb) y2[r0 + j] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// LU solve (split apply, middle kernel, packed-LU factors): y2 = U^-1 L^-1 P y1.
//
// One warp per macro, no CTA barriers: lane l owns rows l and l + 32 of every
// 64-row block.  The packed factor is column-major inside panels and
// triangles (packed_lu.cuh), so per column a warp reads its block rows with
// one coalesced 256-byte access; the block's right-hand side and solution
// stay in the warp's slice of shared memory.  A block step is a panel GEMV
// (sixteen columns of loads in flight per lane) and a substitution with the
// diagonal triangle (column sweep: the final entry broadcast by a shuffle,
// the rows below updated in registers); many warps per SM keep HBM busy while
// each walks its macro's dependent block steps.
// ---------------------------------------------------------------------------
constexpr int LUW_NT = 128;
#ifndef MHDG_LUW_CH
#define MHDG_LUW_CH 8
#endif
constexpr int LUW_CH = MHDG_LUW_CH;  // triangle columns per prefetch chunk

struct LuBlk {
  long long fwd_panel, fwd_diag, bwd_panel, bwd_diag;
  int nb, r0, ncol_fwd, ncol_bwd;
};

// rows lane and lane + 32 of an nb-row column-major panel times x[c0 .. c0 + ncol)
__device__ __forceinline__ void luw_panel(const double* __restrict__ P, int nb, int ncol, const double* x, int lane,
                                          double& a0, double& a1) {
  const bool v0 = lane < nb, v1 = lane + 32 < nb;
  int c = 0;
  for (; c + 16 <= ncol; c += 16) {
    double t0[16], t1[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      t0[k] = v0 ? __ldcs(P + (size_t)(c + k) * nb + lane) : 0.0;
      t1[k] = v1 ? __ldcs(P + (size_t)(c + k) * nb + lane + 32) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double xv = x[c + k];
      a0 += t0[k] * xv;
      a1 += t1[k] * xv;
    }
  }
  for (; c < ncol; ++c) {
    const double xv = x[c];
    if (v0) a0 += __ldcs(P + (size_t)c * nb + lane) * xv;
    if (v1) a1 += __ldcs(P + (size_t)c * nb + lane + 32) * xv;
  }
}

template <class C>
__global__ void __launch_bounds__(LUW_NT) k_lu_warp(int n_mac, const double* __restrict__ F,
                                                    const int* __restrict__ perm, double* __restrict__ work) {
  constexpr int n = C::n, NP = ceven(n), NBLK = (n + PLU_NB - 1) / PLU_NB, NWP = LUW_NT / 32;
  extern __shared__ __align__(16) double smw[];
  __shared__ LuBlk blk[NBLK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < NBLK) {
    const PluOffsets o = plu_offsets(n, tid);
    blk[tid] = LuBlk{o.fwd_panel, o.fwd_diag, o.bwd_panel, o.bwd_diag, o.nb, o.r0, o.ncol_fwd, o.ncol_bwd};
  }
  __syncthreads();
  double* yb = smw + warp * NP;  // solution, logical order
  const long long FS = plu_size(n);
  for (int mac = blockIdx.x * NWP + warp; mac < n_mac; mac += gridDim.x * NWP) {
    const double* y1 = Work<C>::y1(work, mac);
    const int* pm = perm + (size_t)mac * n;
    for (int k = lane; k < n; k += 32) yb[k] = y1[__ldg(pm + k)];  // P y1
    __syncwarp();
    const double* Fm = F + (size_t)mac * FS;
    for (int b = 0; b < NBLK; ++b) {  // forward: y_b = L_bb^-1 (y_b - L[b, :b] y_:b)
      const LuBlk o = blk[b];
      double a0 = 0.0, a1 = 0.0;
      luw_panel(Fm + o.fwd_panel, o.nb, o.ncol_fwd, yb, lane, a0, a1);
      // forward substitution with the unit lower diagonal block: column sweep, the final
      // y_c broadcast from its lane, rows below updated in registers
      double v0 = lane < o.nb ? yb[o.r0 + lane] - a0 : 0.0;
      double v1 = lane + 32 < o.nb ? yb[o.r0 + lane + 32] - a1 : 0.0;
      const double* Tl = Fm + o.fwd_diag;
      {  // columns in chunks of LUW_CH, the next chunk's loads in flight during this one's sweep
        const int nc = o.nb - 1;
        auto ld = [&](int c0, double (&l0)[LUW_CH], double (&l1)[LUW_CH]) {
#pragma unroll
          for (int k = 0; k < LUW_CH; ++k) {
            const int c = c0 + k;
            const double* col = Tl + plu_lo_col(o.nb, c) - c - 1;
            l0[k] = (c < nc && lane > c && lane < o.nb) ? __ldcs(col + lane) : 0.0;
            l1[k] = (c < nc && lane + 32 > c && lane + 32 < o.nb) ? __ldcs(col + lane + 32) : 0.0;
          }
        };
        auto sweep = [&](int c0, const double (&l0)[LUW_CH], const double (&l1)[LUW_CH]) {
#pragma unroll
          for (int k = 0; k < LUW_CH; ++k) {  // column c of L_bb: rows c+1 .. nb-1
            const int c = c0 + k;
            if (c < nc) {
              const double yc = __shfl_sync(MHDG_FULL, c < 32 ? v0 : v1, c & 31);
              v0 -= l0[k] * yc;
              v1 -= l1[k] * yc;
            }
          }
        };
        double pa0[LUW_CH], pa1[LUW_CH], pb0[LUW_CH], pb1[LUW_CH];
        ld(0, pa0, pa1);
        for (int c0 = 0; c0 < nc; c0 += 2 * LUW_CH) {
          ld(c0 + LUW_CH, pb0, pb1);
          sweep(c0, pa0, pa1);
          ld(c0 + 2 * LUW_CH, pa0, pa1);
          sweep(c0 + LUW_CH, pb0, pb1);
        }
      }
      if (lane < o.nb) yb[o.r0 + lane] = v0;
      if (lane + 32 < o.nb) yb[o.r0 + lane + 32] = v1;
      __syncwarp();
    }
    for (int b = NBLK - 1; b >= 0; --b) {  // backward: x_b = U_bb^-1 (y_b - U[b, b+1:] x_b+1:)
      const LuBlk o = blk[b];
      double a0 = 0.0, a1 = 0.0;
      luw_panel(Fm + o.bwd_panel, o.nb, o.ncol_bwd, yb + o.r0 + o.nb, lane, a0, a1);
      double v0 = lane < o.nb ? yb[o.r0 + lane] - a0 : 0.0;
      double v1 = lane + 32 < o.nb ? yb[o.r0 + lane + 32] - a1 : 0.0;
      const double* Tu = Fm + o.bwd_diag;
      {  // columns nb-1 .. 0 in chunks, the next chunk's loads in flight
        auto ld = [&](int c0, double (&u0)[LUW_CH], double (&u1)[LUW_CH]) {
#pragma unroll
          for (int k = 0; k < LUW_CH; ++k) {
            const int c = c0 - k;
            const double* col = Tu + (c >= 0 ? c * (c + 1) / 2 : 0);
            u0[k] = (c >= 0 && lane <= c) ? __ldcs(col + lane) : 0.0;
            u1[k] = (c >= 0 && lane + 32 <= c) ? __ldcs(col + lane + 32) : 0.0;
          }
        };
        auto sweep = [&](int c0, const double (&u0)[LUW_CH], const double (&u1)[LUW_CH]) {
#pragma unroll
          for (int k = 0; k < LUW_CH; ++k) {  // column c of U_bb: rows 0 .. c (diagonal: 1/U_cc)
            const int c = c0 - k;
            if (c >= 0) {
              const double xc = __shfl_sync(MHDG_FULL, c < 32 ? v0 * u0[k] : v1 * u1[k], c & 31);
              if (lane == c) v0 = xc;
              else v0 -= u0[k] * xc;
              if (lane + 32 == c) v1 = xc;
              else v1 -= u1[k] * xc;
            }
          }
        };
        double pa0[LUW_CH], pa1[LUW_CH], pb0[LUW_CH], pb1[LUW_CH];
        ld(o.nb - 1, pa0, pa1);
        for (int c0 = o.nb - 1; c0 >= 0; c0 -= 2 * LUW_CH) {
          ld(c0 - LUW_CH, pb0, pb1);
          sweep(c0, pa0, pa1);
          ld(c0 - 2 * LUW_CH, pa0, pa1);
          sweep(c0 - LUW_CH, pb0, pb1);
        }
      }
      if (lane < o.nb) yb[o.r0 + lane] = v0;
      if (lane + 32 < o.nb) yb[o.r0 + lane + 32] = v1;
      __syncwarp();
    }
    double* y2 = Work<C>::y2(work, n_mac, mac);
    for (int k = lane; k < n; k += 32) y2[k] = yb[k];
    __syncwarp();
  }
}

template <class C>
static int launch_lu_stream(const mhdg_disc& g, const mhdg_factors& f, cudaStream_t st) {
  const size_t bytes = sizeof(double) * (LUW_NT / 32) * ceven(C::n);
  auto kern = k_lu_warp<C>;
  static int ctas = 0;
  if (!ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, LUW_NT, bytes);
    ctas = sms * (per > 0 ? per : 1);
  }
  const int need = (g.n_mac + LUW_NT / 32 - 1) / (LUW_NT / 32);
  const int grid = need < ctas ? need : ctas;
  kern<<<grid, LUW_NT, bytes, st>>>(g.n_mac, f.lu, f.perm, f.work);
  return launch_ok();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int g_stream_grid = 0;
// L2 prefetch lookahead in pieces (0: ring only; < 0: the default, 4 pieces -- measured
// C3 apply 8.41 -> 8.08 ms (8: 8.23, 16: 9.23), C2 2.174 -> 2.155 ms)
static int g_pref_ahead = -1;
extern "C" void mhdg_set_stream_prefetch(int pieces) { g_pref_ahead = pieces; }
extern "C" int mhdg_stream_grid(void) { return g_stream_grid; }

template <class C>
static int count_pieces() {
  Sched<C, 0> sc;
  Piece p;
  int k = 0;
  while (sc.next(p)) ++k;
  return k;
}

// ring stages per kernel (all instantiations run two CTAs per SM; 3D keeps its
// class tables in global memory and the parts' work areas apart to fit)
#ifndef MHDG_STAGES_3D_PRE
#define MHDG_STAGES_3D_PRE 3
#endif
#ifndef MHDG_STAGES_3D_POST
#define MHDG_STAGES_3D_POST 4
#endif
#ifndef MHDG_STAGES_2D_POST
#define MHDG_STAGES_2D_POST 5
#endif
template <class C>
__host__ __device__ constexpr int stages_of(int part) {
  const int dflt = C::D == 2 ? (part == 2 ? MHDG_STAGES_2D_POST : MHDG_STAGES)
                             : (part == 2 ? MHDG_STAGES_3D_POST : (part == 1 ? MHDG_STAGES_3D_PRE : MHDG_STAGES));
  // post part with the resident M^-1 D table: the stages that still fit beside it
  return part == 2 && post_mdr<C>() && post_stages_mdr<C>() < dflt ? post_stages_mdr<C>() : dflt;
}

static int g_split = 1;
extern "C" void mhdg_set_apply_split(int on) { g_split = on; }

template <class C>
static bool stream_ok(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f) {
  static const int npieces = count_pieces<C>();
  if (npieces > maxp_of<C>()) return false;
  if (g.dim != C::D || g.L != C::L || g.Lf != C::LF || g.nloc != C::NLOC || g.nq != C::NQ || g.n_sub != C::NSUB ||
      g.n_tri != C::NTRI || g.nlocf != C::NLOCF || g.nqf != C::NQF)
    return false;
  // 16-byte alignment of every per-macro segment base
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool sizes = ((C::NF * C::BS * C::BS) % 2 == 0) && ((C::NPF * C::NWF) % 2 == 0);  // W_vol: either
  const bool tables = g.n_grad_cls >= 1 && g.grad_cls && g.grad_cls_of && g.node_to_face && g.minv_d_face &&
                      g.n_face_nodes == C::NFN;
  const size_t cls = C::D == 2 ? (size_t)g.n_grad_cls * TSm<C>::CLS : 0;
  const size_t smem = sizeof(double) * ((size_t)stages_of<C>(0) * ST_DBL + SSm<C, 0>::total + TSm<C>::total +
                                        (cls <= (size_t)C::D * C::n ? cls : 2 * cls));
  return sizes && tables && (f.kind == 0 || (f.kind == 1 && f.work && g_split)) && smem <= 227 * 1024 &&
         al(b.face_state_trace) && al(b.face_trace_trace) &&
         al(b.face_trace_state) && al(b.wdgdq_vol) && al(b.wdgdq_face) && al(f.lu) && al(f.work);
}

template <class C, int STAGES, int PART>
static size_t stream_smem(const mhdg_disc& g) {
  // 2D: class tables (+ per-macro gphys unless it fits in z) in shared memory; 3D: none
  const size_t cls = C::D == 2 ? (size_t)g.n_grad_cls * TSm<C>::CLS : 0;
  return sizeof(double) * ((size_t)STAGES * ST_DBL + SSm<C, PART>::total + TSm<C>::total +
                           (PART != 2 ? (cls <= (size_t)C::D * C::n ? cls : 2 * cls)
                                      : (post_mdr<C>() ? (size_t)md_table<C>() : 0)));
}

template <class C, int STAGES, int PART>
static int launch_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x,
                         double* y_loc, cudaStream_t st, StreamIn sin = StreamIn{nullptr, 0.0, nullptr, 0.0}) {
  const size_t bytes = stream_smem<C, STAGES, PART>(g);
  if (bytes > 227 * 1024) return MHDG_ERR_CONFIG;
  auto kern = k_apply_stream<C, STAGES, PART>;
  static int ctas = 0;
  if (!ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NCONS + 32, bytes);
    ctas = sms * (per > 0 ? per : 1);
  }
  const int grid = g.n_mac < ctas ? g.n_mac : ctas;
  g_stream_grid = grid;
  const int pref = g_pref_ahead >= 0 ? g_pref_ahead : 4;
  kern<<<grid, NCONS + 32, bytes, st>>>(g, b, f, x, y_loc, pref, sin);
  return launch_ok();
}

#ifndef MHDG_SI_STAGES
#define MHDG_SI_STAGES 3
#endif
#ifndef MHDG_SI_NCT
#define MHDG_SI_NCT 256
#endif

template <class C>
static int launch_si(const mhdg_disc& g, const mhdg_factors& f, cudaStream_t st) {
  constexpr int STG = MHDG_SI_STAGES, NCT = MHDG_SI_NCT;
  const size_t bytes = sizeof(double) * ((size_t)STG * ST_DBL + ceven(C::n));
  auto kern = k_si_stream<C, STG, NCT>;
  static int ctas = 0;
  if (!ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NCT + 32, bytes);
    ctas = sms * (per > 0 ? per : 1);
  }
  const long long units = (long long)g.n_mac * C::NBLK;
  const int grid = units < ctas ? (int)units : ctas;
  kern<<<grid, NCT + 32, bytes, st>>>(g.n_mac, f.lu, f.work);
  return launch_ok();
}



// split apply: pre (y1, face terms) -> S^-1 stream (y2) -> post (y_loc)
template <class C>
static int launch_apply(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x,
                        double* y_loc, cudaStream_t st) {
  if (!f.work || !g_split) {
    tl_begin(TL_APPLY_FUSED, st);
    const int rc0 = launch_stream<C, stages_of<C>(0), 0>(g, b, f, x, y_loc, st);
    tl_end(TL_APPLY_FUSED, st);
    return rc0;
  }
  tl_begin(TL_APPLY_PRE, st);
  int rc = launch_stream<C, stages_of<C>(1), 1>(g, b, f, x, y_loc, st);
  tl_end(TL_APPLY_PRE, st);
  if (rc) return rc;
  tl_begin(TL_APPLY_SI, st);
  rc = f.kind == 1 ? launch_lu_stream<C>(g, f, st) : launch_si<C>(g, f, st);
  tl_end(TL_APPLY_SI, st);
  if (rc) return rc;
  tl_begin(TL_APPLY_POST, st);
  rc = launch_stream<C, stages_of<C>(2), 2>(g, b, f, x, y_loc, st);
  tl_end(TL_APPLY_POST, st);
  return rc;
}

#ifdef MHDG_STREAM_PROFILE
extern "C" int mhdg_stream_profile(unsigned long long* out, int reset) {
  if (out) cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    unsigned long long z[16][3] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  }
  return 0;
}
#endif

template <int D> int mass_solve_all(const mhdg_disc&, const double*, double*, cudaStream_t);
template <int D> int recover_dq(const mhdg_disc&, const double*, const double*, const double*, long long, double*,
                                double*, cudaStream_t);

// Condensed rhs and recovery (condense.py:105-127) on the split apply's kernels:
//   rhs:      zr = A_qq^-1 R_Q; pre with x = 0, z = -zr, y1 + R_U  -> t2 = S^-1 (R_U - A_uq zr)
//             -> post: b_loc = A_hu t2 - A_hq A_qq^-1 A_qu t2 + A_hq zr;
//   recover:  zr; pre with x = dtrace, z += zr, y1 - R_U -> du = S^-1 (A_uq zr - R_U + y1(dtrace))
//             -> k_recover_dq: dq = -zr - A_qq^-1 A_qu du - A_qq^-1 A_qh dtrace.
// zr lives in the factors' Schur scratch (dead after the factorization).
template <class C>
static int cond_stream_impl(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, bool rhs,
                            const double* Rg, const double* Ru, const double* dtrace, double* y_loc, double* du,
                            double* dq, cudaStream_t st) {
  double* zr = f.scratch;
  int rc = mass_solve_all<C::D>(g, Rg, zr, st);
  if (rc) return rc;
  const StreamIn sin = rhs ? StreamIn{zr, -1.0, Ru, 1.0} : StreamIn{zr, 1.0, Ru, -1.0};
  tl_begin(TL_APPLY_PRE, st);
  rc = launch_stream<C, stages_of<C>(1), 1>(g, b, f, rhs ? nullptr : dtrace, y_loc, st, sin);
  tl_end(TL_APPLY_PRE, st);
  if (rc) return rc;
  tl_begin(TL_APPLY_SI, st);
  rc = launch_lu_stream<C>(g, f, st);
  tl_end(TL_APPLY_SI, st);
  if (rc) return rc;
  if (rhs) {
    tl_begin(TL_APPLY_POST, st);
    rc = launch_stream<C, stages_of<C>(2), 2>(g, b, f, nullptr, y_loc, st);
    tl_end(TL_APPLY_POST, st);
    return rc;
  }
  return recover_dq<C::D>(g, dtrace, zr, Work<C>::y2(f.work, g.n_mac, 0), (long long)Work<C>::PER, du, dq, st);
}

// -1 when no streamed instantiation matches or the scratch cannot hold zr (generic kernels)
int cond_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, bool rhs, const double* Rg,
                const double* Ru, const double* dtrace, double* y_loc, double* du, double* dq, cudaStream_t st) {
  if (f.kind != 1 || !f.work || !f.scratch || !g_split) return -1;
  const long long n = (long long)g.L * g.ns;
  const long long cap = (f.scratch_macros > 0 && f.scratch_macros < g.n_mac ? f.scratch_macros : g.n_mac) * n * n;
  if (cap < (long long)g.n_mac * g.dim * n) return -1;
#define MHDG_COND(D_, M_, P_) \
  if (stream_ok<Cfg<D_, M_, P_>>(g, b, f)) return cond_stream_impl<Cfg<D_, M_, P_>>(g, b, f, rhs, Rg, Ru, dtrace, y_loc, du, dq, st);
  MHDG_COND(2, 4, 3)
  MHDG_COND(2, 2, 2)
  MHDG_COND(3, 2, 2)
  MHDG_COND(3, 1, 2)
  MHDG_COND(3, 2, 1)
  MHDG_COND(3, 1, 1)
  MHDG_COND(3, 1, 3)
  MHDG_COND(3, 4, 1)
  MHDG_COND(3, 2, 3)
#undef MHDG_COND
  return -1;
}

// returns -1 when no streamed instantiation matches (caller uses k_apply_local)
int apply_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x, double* y_loc,
                 cudaStream_t st) {
  if (stream_ok<Cfg<2, 4, 3>>(g, b, f)) return launch_apply<Cfg<2, 4, 3>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<2, 2, 2>>(g, b, f)) return launch_apply<Cfg<2, 2, 2>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 2, 2>>(g, b, f)) return launch_apply<Cfg<3, 2, 2>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 1, 2>>(g, b, f)) return launch_apply<Cfg<3, 1, 2>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 2, 1>>(g, b, f)) return launch_apply<Cfg<3, 2, 1>>(g, b, f, x, y_loc, st);
  // the rest of the C5 (m, p) sweep (BASELINE configs[4])
  if (stream_ok<Cfg<3, 1, 1>>(g, b, f)) return launch_apply<Cfg<3, 1, 1>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 1, 3>>(g, b, f)) return launch_apply<Cfg<3, 1, 3>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 4, 1>>(g, b, f)) return launch_apply<Cfg<3, 4, 1>>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 2, 3>>(g, b, f)) return launch_apply<Cfg<3, 2, 3>>(g, b, f, x, y_loc, st);
  return -1;
}

}  // namespace mhdg
