// K3: backward of rasterize_meshes on sm_100a (rasterize_backward, MR:329-403, per-slot part MR:345-378).
//
// One thread per fragment slot recomputes the slot's NDC triangle and pixel centre, pulls the cotangents on
// zbuf / bary / dists back through z-interpolation, clamp+renormalise, (optional) perspective correction,
// the barycentric quotient and the frozen-edge distance envelope, and produces the 9 cotangents of its
// face's (x_ndc, y_ndc, z_view) x 3 vertices; empty slots are compacted away first (ballot queue). Lanes of a
// warp that hit the same face (neighbouring pixels
// very often do) are grouped with __match_any_sync and summed with a log-depth shuffle reduction, so ONE
// lane issues the 9 fp64 atomicAdds per (warp, face) instead of one per slot. The reference reduces per
// vertex in slot order on one thread (MR:380-392); here the order of fp64 additions is not fixed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "raster_kernels.cuh"
#include "raster_math.cuh"

namespace drb {

// MR:309-325 (clamp_barycentric_backward)
__device__ __forceinline__ void clamp_bary_backward(const double wr[3], const double dc[3], double out[3]) {
  double t0 = clamp01(wr[0]), t1 = clamp01(wr[1]), t2 = clamp01(wr[2]);
  double s = t0 + t1 + t2;
  if (s <= 0) {
    out[0] = out[1] = out[2] = 0.0;
    return;
  }
  const double rs = fdiv(1.0, s);  // tolerance path: fast reciprocal (raster_math.cuh fdiv)
  double h0 = t0 * rs, h1 = t1 * rs, h2 = t2 * rs;
  double d = dc[0] * h0 + dc[1] * h1 + dc[2] * h2;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double d_t = (dc[i] - d) * rs;
    out[i] = (wr[i] > 0.0 && wr[i] < 1.0) ? d_t : 0.0;
  }
}

// one occupied slot's per-slot inputs (bary + cotangents + the face's face_verts), loaded one batch ahead of
// their use
template <typename InT>
struct SlotIn {
  InT w[3], dz, db[3], dd;
  double v[9];  // the face's face_verts
};
template <typename InT>
__device__ __forceinline__ void load_slot(const BwdArgs<InT>& A, int64_t slot, int32_t fid, SlotIn<InT>& in) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    in.w[k] = __ldcs(A.bary + 3 * slot + k);  // every input is read exactly once: evict-first
    in.db[k] = __ldcs(A.d_bary + 3 * slot + k);
  }
  in.dz = __ldcs(A.d_zbuf + slot);
  in.dd = __ldcs(A.d_dists + slot);
  const double* q = A.fv + 9 * (int64_t)fid;
#pragma unroll
  for (int k = 0; k < 9; ++k) in.v[k] = __ldg(q + k);
}

// per-slot cotangents -> g[9] = (dx, dy, dz) for vertices a, b, c; p = the slot's pixel centre (MR:357)
// kInternalW: the clamped barycentrics used by the z-interpolation term are derived here from the recomputed
// weights (and returned in w_out) instead of being read from the forward's bary output (fused consumers)
// kPC / kCL: perspective_correct / clip_barycentric_coords fixed at compile time (0 / 1), or read from A (2): the
// fixed instantiations carry only their own branch of the chain (smaller code: K3 is instruction-cache sensitive)
template <typename InT, bool kInternalW = false, int kPC = 2, int kCL = 2>
__device__ __forceinline__ void slot_backward(const BwdArgs<InT>& A, V2 p, int32_t fid, const SlotIn<InT>& in,
                                              double g[9], double* w_out = nullptr) {
  const bool persp = kPC == 2 ? A.persp : kPC == 1, clip = kCL == 2 ? A.clip : kCL == 1;
  const FaceGeom fg = make_face_geom(in.v);
  const double z[3] = {fg.z0, fg.z1, fg.z2};

  double w_hat[3] = {(double)in.w[0], (double)in.w[1], (double)in.w[2]};
  const double dz = (double)in.dz;
  // MR:363-365: cotangent on the clamped bary = direct input + z-interpolation path
  const double d_hat[3] = {(double)in.db[0] + dz * z[0], (double)in.db[1] + dz * z[1], (double)in.db[2] + dz * z[2]};
  const V2 pa = p - fg.a, pb = p - fg.b, pc = p - fg.c;
  double w_raw[3];
  barycentric<false>(fg, pa, pb, pc, w_raw);  // MR:366
  double d_w[3], dzv[3] = {0.0, 0.0, 0.0};
  if constexpr (kInternalW) {  // w_hat = the forward's bary: clamp(persp(w_raw)) / clamp(w_raw) (MR:172)
    double u[3];
    if (persp) {
      persp_correct<false>(w_raw, fg.z0, fg.z1, fg.z2, u);
    } else {
      u[0] = w_raw[0];
      u[1] = w_raw[1];
      u[2] = w_raw[2];
    }
    if (clip) {
      clamp_barycentric<false>(u, w_hat);
    } else {
      w_hat[0] = u[0];
      w_hat[1] = u[1];
      w_hat[2] = u[2];
    }
    w_out[0] = w_hat[0];
    w_out[1] = w_hat[1];
    w_out[2] = w_hat[2];
  }
  if (persp) {  // builder-defined: u = persp_correct(w_raw, z); bary = clamp(u)
    double u[3], d_u[3], d_top[3];
    const double den = persp_correct<false>(w_raw, fg.z0, fg.z1, fg.z2, u);
    if (clip) {
      clamp_bary_backward(u, d_hat, d_u);
    } else {
      d_u[0] = d_hat[0];
      d_u[1] = d_hat[1];
      d_u[2] = d_hat[2];
    }
    if (den > kPerspEps) {
      const double rden = fdiv(1.0, den);
      const double du_u = d_u[0] * u[0] + d_u[1] * u[1] + d_u[2] * u[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) d_top[k] = (d_u[k] - du_u) * rden;
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) d_top[k] = d_u[k] * (1.0 / kPerspEps);
    }
    d_w[0] = d_top[0] * z[1] * z[2];
    d_w[1] = d_top[1] * z[0] * z[2];
    d_w[2] = d_top[2] * z[0] * z[1];
    dzv[0] = d_top[1] * w_raw[1] * z[2] + d_top[2] * w_raw[2] * z[1];
    dzv[1] = d_top[0] * w_raw[0] * z[2] + d_top[2] * w_raw[2] * z[0];
    dzv[2] = d_top[0] * w_raw[0] * z[1] + d_top[1] * w_raw[1] * z[0];
  } else if (clip) {
    clamp_bary_backward(w_raw, d_hat, d_w);  // MR:367
  } else {
    d_w[0] = d_hat[0];
    d_w[1] = d_hat[1];
    d_w[2] = d_hat[2];
  }

  // MR:290-306 barycentric_backward (w recomputed there == w_raw)
  const V2 a = fg.a, b = fg.b, c = fg.c;
  const V2 grad_d_a = perp(b - c), grad_d_b = perp(c - a), grad_d_c = perp(a - b);
  const V2 gn0_b = perp(c - p), gn0_c = perp(p - b);
  const V2 gn1_c = perp(a - p), gn1_a = perp(p - c);
  const V2 gn2_a = perp(b - p), gn2_b = perp(p - a);
  const double inv = fdiv(1.0, fg.area);
  const double wd = w_raw[0] * d_w[0] + w_raw[1] * d_w[1] + w_raw[2] * d_w[2];
  V2 dxy[3];
  dxy[0] = ((gn1_a * d_w[1] + gn2_a * d_w[2]) - grad_d_a * wd) * inv;
  dxy[1] = ((gn0_b * d_w[0] + gn2_b * d_w[2]) - grad_d_b * wd) * inv;
  dxy[2] = ((gn0_c * d_w[0] + gn1_c * d_w[1]) - grad_d_c * wd) * inv;

  // MR:46-69 point_triangle_dist2_backward: nearest edge (first strict min), t and sign frozen
  const double d_out = (double)in.dd;
  // the nearest point of each edge (the same expressions seg_dist2 evaluates), carried through the argmin instead
  // of re-selecting the edge's endpoints afterwards
  const double t0 = seg_t<false>(dot(pa, fg.ab), fg.len_ab), t1 = seg_t<false>(dot(pb, fg.bc), fg.len_bc),
               t2 = seg_t<false>(dot(pc, fg.ca), fg.len_ca);
  const V2 q0 = a + fg.ab * t0, q1 = b + fg.bc * t1, q2 = c + fg.ca * t2;
  const double e0 = norm2(p - q0), e1 = norm2(p - q1), e2 = norm2(p - q2);
  int be = 0;
  double best = e0, bt = t0;
  V2 qq = q0;
  if (e1 < best) { best = e1; bt = t1; be = 1; qq = q1; }
  if (e2 < best) { best = e2; bt = t2; be = 2; qq = q2; }
  const bool inside = point_triangle_dist2<false>(p, fg, pa, pb, pc).inside;
  const double sign = inside ? -1.0 : 1.0;
  const V2 gg = (qq - p) * (2.0 * sign * d_out);
  const V2 g_first = gg * (1.0 - bt), g_second = gg * bt;
  // grads[be] += g*(1-t); grads[(be+1)%3] += g*t
  if (be == 0) { dxy[0] = dxy[0] + g_first; dxy[1] = dxy[1] + g_second; }
  else if (be == 1) { dxy[1] = dxy[1] + g_first; dxy[2] = dxy[2] + g_second; }
  else { dxy[2] = dxy[2] + g_first; dxy[0] = dxy[0] + g_second; }

#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g[3 * k + 0] = dxy[k].x;
    g[3 * k + 1] = dxy[k].y;
    g[3 * k + 2] = dz * w_hat[k] + dzv[k];  // MR:375
  }
}

// Sum g[NV] over the lanes of each __match_any_sync(fid) group (log-depth shuffle tree); returns true on the
// group's lowest lane, which then owns the group total.
template <int NV = 9>
__device__ __forceinline__ bool reduce_by_face(int32_t fid, int lane, double g[NV]) {
  const int key = fid >= 0 ? fid : -1 - lane;  // inactive lanes form singleton groups that never write
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  unsigned rel = __popc(peers & ((1u << lane) - 1u));
  unsigned rem = peers & ~((2u << lane) - 1u);  // peers above this lane (2u << 31 == 0)
  while (__any_sync(0xffffffffu, rem != 0)) {
    const int next = __ffs(rem);  // 1-based lane of the next peer, 0 if none
    const int src = next ? next - 1 : lane;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double t = __shfl_sync(0xffffffffu, g[k], src);
      if (next) g[k] += t;
    }
    rem &= ~__ballot_sync(0xffffffffu, rel & 1u);
    rel >>= 1;
  }
  return fid >= 0 && (peers & ((1u << lane) - 1u)) == 0;
}

// Persistent warps walk the slots in chunks of kChunk consecutive slots. Occupied slots (pix_to_face >= 0;
// typically 40-70 % of them) are compacted with ballot + popc into a warp-private queue and processed 32 at
// a time, so every lane of a batch does a full per-slot backward.
constexpr int kBwdChunk = 32 * 16;
constexpr int kBwdMinBlocks = 4;
// 128-thread CTAs, 4 per SM (128 registers, no spills since the (perspective_correct, clip) instantiations; C4
// 2.44 -> 2.29 ms against 3 per SM at 155 registers). Round 1: 80 registers x 24 warps 3.47 ms, 96 x 20 3.33 ms,
// 128 x 16 3.10 ms with the first design; with the prefetching one 128 x 16 (36-byte spills) 2.54 ms, 155 x 12
// 2.48 ms (profiles/r01/README.md, profiles/r02/README.md).
constexpr int kBwdThreads = 128;

template <typename InT, int kPC, int kCL>
__device__ __forceinline__ void backward_batch(const BwdArgs<InT>& A, V2 p, int32_t my_fid, const SlotIn<InT>& in,
                                               int lane) {
  double g[9];
  if (my_fid >= 0) {
    slot_backward<InT, false, kPC, kCL>(A, p, my_fid, in, g);
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) g[k] = 0.0;
  }
  if (reduce_by_face(my_fid, lane, g)) {
    double* out = A.grad + 9 * (int64_t)my_fid;
#pragma unroll
    for (int k = 0; k < 9; ++k) atomicAdd(out + k, g[k]);
  }
}

// Phase A: the warp loads its whole 512-slot chunk of pix_to_face at once (16 independent coalesced loads per
// lane in flight, instead of one exposed load latency per 32 slots) and compacts the occupied slots into a
// warp-private queue in shared memory. Phase B: the queue is processed 32 slots per step, the next step's
// bary / cotangents loaded before the current step computes.
constexpr int kPixTab = 2048;  // pixel-centre tables in shared memory when H + W fits

constexpr int kBwdMaxChunksPerCta = 32;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <typename InT, int kPC, int kCL>
__device__ __forceinline__ void backward_chunk(const BwdArgs<InT>& A, int64_t c0, int n, const uint16_t* qo,
                                               const int32_t* qf, const double* pix_tab, bool tab, int lane) {
  const int HW = A.H * A.W;
  // slot -> pixel with one 64-bit division per chunk; 32-bit arithmetic per slot
  const int64_t pix0 = c0 / A.K;
  const int r0 = (int)(c0 - pix0 * A.K);
  const int pp0 = (int)(pix0 % HW);
  SlotIn<InT> nxt;
  int32_t nfid = -1;
  int noff = 0;
  if (lane < n) {
    noff = qo[lane];
    nfid = qf[lane];
    load_slot(A, c0 + noff, nfid, nxt);
  }
  for (int q0 = 0; q0 < n; q0 += 32) {
    const SlotIn<InT> cur = nxt;
    const int32_t my_fid = nfid;
    const int off = noff;
    nfid = -1;
    if (q0 + 32 + lane < n) {
      noff = qo[q0 + 32 + lane];
      nfid = qf[q0 + 32 + lane];
      load_slot(A, c0 + noff, nfid, nxt);
    }
    V2 p{0.0, 0.0};
    if (my_fid >= 0) {
      uint32_t pp = (uint32_t)pp0 + A.divK.div((uint32_t)(r0 + off));
      if (pp >= (uint32_t)HW) pp %= (uint32_t)HW;  // the chunk crossed into the next image
      const uint32_t i = A.divW.div(pp), j = pp - i * (uint32_t)A.W;
      p = tab ? V2{pix_tab[j], pix_tab[A.W + i]} : V2{pixel_x(A.W, (int)j), pixel_y(A.H, (int)i)};  // MR:357
    }
    backward_batch<InT, kPC, kCL>(A, p, my_fid, cur, lane);
  }
}

// CTA = A.cpc consecutive chunks; its warps take chunks from a shared counter (so they finish
// together and the CTA's registers are released without idle warps holding them). While a warp computes chunk
// c, the pix_to_face words of its next chunk stream into shared memory with cp.async (no registers held);
// the chunk is then compacted (occupied slots -> queue of 16-bit offsets + face ids) straight from shared memory.
template <typename InT, int kPC, int kCL>
__global__ void __launch_bounds__(kBwdThreads, kBwdMinBlocks) k_backward(BwdArgs<InT> A) {
  constexpr int NWB = kBwdThreads / 32;
  __shared__ __align__(16) int64_t stage[NWB][kBwdChunk];
  __shared__ int32_t q_fid[NWB][kBwdChunk];
  __shared__ uint16_t q_off[NWB][kBwdChunk];
  __shared__ double pix_tab[kPixTab];  // pixel_x(W, j) for j < W, then pixel_y(H, i) (camera.cpp:100-102)
  __shared__ int next_chunk;
  const bool tab = A.W + A.H <= kPixTab;
  if (threadIdx.x == 0) next_chunk = NWB;  // chunk w is warp w's first
  if (tab)
    for (int t = threadIdx.x; t < A.W + A.H; t += kBwdThreads)
      pix_tab[t] = t < A.W ? pixel_x(A.W, t) : pixel_y(A.H, t - A.W);
  __syncthreads();
  constexpr int kSteps = kBwdChunk / 32;
  // chunk k of this CTA starts at slot chunk0(k); valid while k < A.cpc and it starts before S
  // (only k is carried across the chunk's compute: everything else is recomputed, to stay spill-free)
  auto chunk0 = [&](int k) {
    return ((int64_t)blockIdx.x * A.cpc + k) * kBwdChunk;
  };
  auto valid = [&](int k) { return k < A.cpc && chunk0(k) < A.S; };
  auto issue = [&](int k) {  // start the copy of chunk k's pix_to_face words (slots past S are not copied)
    const int lane = threadIdx.x & 31;
    const int64_t c0 = chunk0(k);
    int64_t* stg = stage[threadIdx.x >> 5];
#pragma unroll
    for (int t = 0; t < kSteps; ++t) {
      const int64_t slot = c0 + t * 32 + lane;
      if (slot < A.S) cp_async8(stg + t * 32 + lane, A.p2f + slot);
    }
    cp_async_commit();
  };
  int k = threadIdx.x >> 5;
  if (valid(k)) issue(k);
  while (valid(k)) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c0 = chunk0(k);
    const int64_t* stg = stage[wid];
    uint16_t* qo = q_off[wid];
    int32_t* qf = q_fid[wid];
    cp_async_wait_all();
    __syncwarp();
    int n = 0;
    // (a rank-major queue order, which merges more same-face lanes per reduce_by_face, measured slower: C4 2.48 ->
    // 3.05 ms, longer reductions and scattered input loads)
#pragma unroll 4
    for (int t = 0; t < kSteps; ++t) {
      const int o = t * 32 + lane;
      const int64_t slot = c0 + o;
      const int64_t f = slot < A.S ? stg[o] : -1;
      const bool occ = f >= 0 && f < A.F;
      const unsigned m = __ballot_sync(0xffffffffu, occ);
      if (occ) {
        const int pos = n + __popc(m & ((1u << lane) - 1u));
        qo[pos] = (uint16_t)o;
        qf[pos] = (int32_t)f;
      }
      n += __popc(m);
    }
    __syncwarp();
    int kn = 0;
    if (lane == 0) kn = atomicAdd(&next_chunk, 1);
    kn = __shfl_sync(0xffffffffu, kn, 0);
    if (valid(kn)) issue(kn);  // overlaps this chunk's compute
    backward_chunk<InT, kPC, kCL>(A, c0, n, qo, qf, pix_tab, A.W + A.H <= kPixTab, lane);
    __syncwarp();
    k = kn;
  }
}

// ------------------------------------------------------------------------------------------------
// Fused silhouette backward: silhouette_blend_backward (shading.cpp:93-121) feeding rasterize_backward
// (MR:329-403) with d_zbuf = d_bary = 0, as the reference's fit loop calls them (pipeline.cpp:153-162). Only
// the distance envelope (MR:46-69) carries gradient, so the per-slot work is: recompute the slot's signed
// distance, d_dist = d_alpha * prod_{other occupied slots}(1 - prob) * (-prob (1 - prob) / sigma), and push it
// through the frozen nearest edge. One lane per pixel walks its K slots three times: probabilities (into
// shared memory), suffix products, then prefix products + gradients; lanes stay in step over s so the
// gradients of one s are summed per face across the warp (reduce_by_face) before the atomics. The product over
// the other slots is prefix * suffix instead of the reference's left-to-right loop (different rounding, same
// value within the 1e-4 gradient tolerance); fragments and their cotangents never touch HBM.

__device__ __forceinline__ void silhouette_envelope(const double* v, V2 p, double& dist, int& be, double& bt, V2& qq,
                                                    double& sign) {
  const FaceGeom fg = make_face_geom(v);
  const V2 pa = p - fg.a, pb = p - fg.b, pc = p - fg.c;
  // as slot_backward: each edge's nearest point carried through the argmin
  const double t0 = seg_t<false>(dot(pa, fg.ab), fg.len_ab), t1 = seg_t<false>(dot(pb, fg.bc), fg.len_bc),
               t2 = seg_t<false>(dot(pc, fg.ca), fg.len_ca);
  const V2 q0 = fg.a + fg.ab * t0, q1 = fg.b + fg.bc * t1, q2 = fg.c + fg.ca * t2;
  const double e0 = norm2(p - q0), e1 = norm2(p - q1), e2 = norm2(p - q2);
  be = 0;
  double best = e0;
  bt = t0;
  qq = q0;
  if (e1 < best) { best = e1; bt = t1; be = 1; qq = q1; }
  if (e2 < best) { best = e2; bt = t2; be = 2; qq = q2; }
  const bool inside = point_triangle_dist2<false>(p, fg, pa, pb, pc).inside;
  sign = inside ? -1.0 : 1.0;
  dist = inside ? -best : best;
}

constexpr int kSilThreads = 128;
constexpr int kSilStoreMaxK = 16;  // up to this K the pass-1 envelope is kept in shared memory for pass 3

// kStore: pass 1 keeps each slot's distance envelope ((qq - p) * 2 sign, t, nearest edge) in shared memory, so
// pass 3 needs no second geometry evaluation (K <= kSilStoreMaxK); otherwise pass 3 recomputes it.
template <bool kStore>
__global__ void __launch_bounds__(kSilThreads) k_silhouette_backward(SilBwdArgs A) {
  // 1 / sigma once (products instead of per-slot divisions; the opacities are tolerance values)
  const double inv_sigma = 1.0 / A.sigma;
  extern __shared__ double sil_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int K = A.K;
  const size_t per_warp = (size_t)K * 32 * (kStore ? 5 : 2) + (size_t)K * 16 * (kStore ? 2 : 1);  // doubles
  double* P = sil_smem + (size_t)wid * per_warp;  // [K][32] prob (-1: empty)
  double* Sf = P + K * 32;     // [K][32] prod_{s2 > s} (1 - prob)
  double* EX = Sf + K * 32;    // [K][32] (qq - p).x * 2 sign      (kStore)
  double* EY = EX + K * 32;    // [K][32] (qq - p).y * 2 sign      (kStore)
  double* BT = EY + K * 32;    // [K][32] t on the nearest edge    (kStore)
  int* BE = reinterpret_cast<int*>(BT + K * 32);  // [K][32] nearest edge (kStore)
  // [32][K] the warp's pix_to_face block (32 consecutive pixels x K slots: one contiguous, coalesced load)
  int32_t* FID = kStore ? BE + K * 32 : reinterpret_cast<int32_t*>(Sf + K * 32);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t HW = (int64_t)A.H * A.W;
  for (int64_t base = warp * 32; base < A.npix; base += nwarps * 32) {
    const int64_t pix = base + lane;
    const double da = pix < A.npix ? (A.d_alpha64 ? A.d_alpha64[pix] : (double)A.d_alpha[pix]) : 0.0;
    const bool act = da != 0.0;  // shading.cpp:102: pixels with d_alpha == 0 contribute nothing
    if (!__any_sync(0xffffffffu, act)) continue;
    const int rem = act ? (int)(pix % HW) : 0;
    const int i = rem / A.W, j = rem - (rem / A.W) * A.W;
    const V2 p{pixel_x(A.W, j), pixel_y(A.H, i)};
    {  // coalesced, 8 loads in flight per lane
      const int64_t n = (A.npix - base < 32 ? A.npix - base : 32) * K;
      const int64_t* src = A.p2f + base * K;
      for (int t0 = 0; t0 < 32 * K; t0 += 256) {
        int64_t f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * 32 + lane;
          f[u] = t < n && t < 32 * K ? __ldcs(src + t) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * 32 + lane;
          if (t < 32 * K) FID[t] = (f[u] >= 0 && f[u] < A.F) ? (int32_t)f[u] : -1;
        }
      }
      __syncwarp();
    }
    const int32_t* row = FID + lane * K;
    // pass 1: per-slot probabilities (and the envelope); the next occupied slot's face_verts are loaded while
    // the current slot is evaluated
    double vn[9];
    int32_t fn = act ? row[0] : -1;
    if (fn >= 0) {
#pragma unroll
      for (int t = 0; t < 9; ++t) vn[t] = __ldg(A.fv + 9 * (int64_t)fn + t);
    }
    for (int s = 0; s < K; ++s) {
      double prob = -1.0;
      const int32_t f = fn;
      double v[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) v[t] = vn[t];
      fn = (act && s + 1 < K) ? row[s + 1] : -1;
      if (fn >= 0) {
#pragma unroll
        for (int t = 0; t < 9; ++t) vn[t] = __ldg(A.fv + 9 * (int64_t)fn + t);
      }
      if (act) {
        if (f >= 0) {
          double dist, bt, sign;
          int be;
          V2 qq;
          silhouette_envelope(v, p, dist, be, bt, qq, sign);
          // sigmoid(-dist / sigma) (shading.cpp:9, 82); fp32 exp for the fp32 cotangent (the value enters the
          // gradients within tolerance), fp64 exp for the fp64 one
          prob = A.d_alpha64 ? fdiv(1.0, 1.0 + exp(dist * inv_sigma))
                             : fdiv(1.0, 1.0 + (double)expf((float)(dist * inv_sigma)));
          if constexpr (kStore) {
            EX[s * 32 + lane] = (qq.x - p.x) * (2.0 * sign);
            EY[s * 32 + lane] = (qq.y - p.y) * (2.0 * sign);
            BT[s * 32 + lane] = bt;
            BE[s * 32 + lane] = be;
          }
        }
      }
      P[s * 32 + lane] = prob;
    }
    // pass 2: suffix products
    double suf = 1.0;
    for (int s = K - 1; s >= 0; --s) {
      Sf[s * 32 + lane] = suf;
      const double pr = P[s * 32 + lane];
      if (pr >= 0.0) suf *= 1.0 - pr;
    }
    // pass 3: d_dists (shading.cpp:115-117) and the distance envelope (MR:46-69) per slot
    double pre = 1.0;
    for (int s = 0; s < K; ++s) {
      const double pr = P[s * 32 + lane];
      int32_t fid = -1;
      double g[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (pr >= 0.0) {
        fid = row[s];
        double ex, ey, bt;
        int be;
        if constexpr (kStore) {
          ex = EX[s * 32 + lane];
          ey = EY[s * 32 + lane];
          bt = BT[s * 32 + lane];
          be = BE[s * 32 + lane];
        } else {
          double v[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) v[t] = __ldg(A.fv + 9 * (int64_t)fid + t);
          double dist, sign;
          V2 qq;
          silhouette_envelope(v, p, dist, be, bt, qq, sign);
          ex = (qq.x - p.x) * (2.0 * sign);
          ey = (qq.y - p.y) * (2.0 * sign);
        }
        const double rest = pre * Sf[s * 32 + lane];
        const double d_out = da * rest * (-pr * (1.0 - pr) * inv_sigma);
        const V2 gg{ex * d_out, ey * d_out};  // (qq - p) * (2 sign d_out): the same single rounding
        const V2 g_first = gg * (1.0 - bt), g_second = gg * bt;
        const int v0 = be, v1 = be == 2 ? 0 : be + 1;
        g[2 * v0] += g_first.x;
        g[2 * v0 + 1] += g_first.y;
        g[2 * v1] += g_second.x;
        g[2 * v1 + 1] += g_second.y;
        pre *= 1.0 - pr;
      }
      if (reduce_by_face<6>(fid, lane, g)) {
        double* out = A.grad + 9 * (int64_t)fid;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          atomicAdd(out + 3 * k, g[2 * k]);
          atomicAdd(out + 3 * k + 1, g[2 * k + 1]);
        }
      }
    }
  }
}

// Slot-compacted variant (K <= kSilQMaxK): the warp's 32 pixels x K slots are compacted to their occupied
// slots, and the two geometry passes run lane-per-SLOT, 32 occupied slots per step (as K3), instead of
// lane-per-pixel walks where a pixel with few candidates idles its lane while a busy neighbour works:
//   A  pix_to_face block + d_alpha + pixel centres -> shared memory; the occupied slots of active pixels -> queue
//   B  per queued slot: distance envelope + prob = sigmoid(-dist / sigma)          (lane per slot)
//   C  per pixel: suffix products, then coefficient da * prefix * suffix * dprob   (lane per pixel, K steps)
//   D  per queued slot: the envelope gradient, reduce_by_face, fp64 atomics       (lane per slot)
constexpr int kSilQMaxK = 64;
constexpr int kSilQWarps = 1;  // one-warp CTAs: 14 resident per SM by shared memory (C4: 4 warps 3.65 ms, 2 3.11, 1 2.87)

// chunk size: at most 256 slots and 28 pixels (shared memory per warp sets the resident warps: measured C4 (K=8)
// 28 px 2.54 ms vs 32 px 2.73, 24 px 2.60, 16 px 2.78; C5 (K=50) 5 px 2.80 vs 10 px 3.55, 3 px 2.98)
constexpr int kSilQSlots = 256, kSilQMaxP = 28;
__host__ __device__ __forceinline__ int silq_pixels(int K) {
  return K >= kSilQSlots ? 1 : min(kSilQMaxP, kSilQSlots / K);
}
__host__ __device__ __forceinline__ size_t silq_warp_bytes(int K) {
  const size_t n = (size_t)silq_pixels(K) * K;
  return n * (5 * sizeof(double) + sizeof(int64_t) + sizeof(int32_t) + sizeof(int32_t) + sizeof(uint16_t)) +
         32 * 4 * sizeof(double) + 8;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// kK: K fixed at compile time (8, the headline K: constant chunk layout and slot -> pixel divisions), 0 = from A
template <int kK = 0>
__global__ void __launch_bounds__(kSilQWarps * 32) k_silhouette_backward_q(SilBwdArgs A) {
  // 1 / sigma once (products instead of per-slot divisions; the opacities are tolerance values)
  const double inv_sigma = 1.0 / A.sigma;
  extern __shared__ double silq_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int K = kK ? kK : A.K;
  const int KS = K;  // per-pixel row stride (K + 1, conflict-free for the lane-per-pixel pass, measured slower)
  const int P = silq_pixels(K);
  const int n = P * KS;
  unsigned char* wb = reinterpret_cast<unsigned char*>(silq_smem) + (size_t)wid * silq_warp_bytes(K);
  double* PR = reinterpret_cast<double*>(wb);  // [n] prob (-1: empty / inactive)
  double* EX = PR + n;                          // [n] (qq - p).x * 2 sign
  double* EY = EX + n;                          // [n] (qq - p).y * 2 sign
  double* BT = EY + n;                          // [n] t on the nearest edge
  double* CO = BT + n;                          // [n] suffix products, then the d_dist coefficient
  double* PXY = CO + n;                         // [32][2] pixel centres
  double* DAS = PXY + 64;                       // [32] staged d_alpha of the next chunk (fp32 or fp64 bits)
  int64_t* STG = reinterpret_cast<int64_t*>(DAS + 32);  // [n] staged pix_to_face of the next chunk
  int32_t* FID = reinterpret_cast<int32_t*>(STG + n);   // [n] face id per slot (-1: empty)
  int32_t* BE = FID + n;                                // [n] nearest edge
  uint16_t* Q = reinterpret_cast<uint16_t*>(BE + n);    // [n] queued slot offsets
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t HW = (int64_t)A.H * A.W;
  // the next chunk's pix_to_face block and d_alpha stream into shared memory (cp.async) while this one computes
  auto issue = [&](int64_t b0) {
    const int64_t pix = b0 + lane;
    if (lane < P && pix < A.npix) {
      if (A.d_alpha64) cp_async8(DAS + lane, A.d_alpha64 + pix);
      else cp_async4(reinterpret_cast<float*>(DAS) + lane, A.d_alpha + pix);
    }
    const int64_t ns = (A.npix - b0 < P ? A.npix - b0 : P) * K;
    for (int t = lane; t < ns; t += 32) cp_async8(STG + t, A.p2f + b0 * K + t);
    cp_async_commit();
  };
  if (warp * P < A.npix) issue(warp * P);
  for (int64_t base = warp * P; base < A.npix; base += nwarps * P) {
    cp_async_wait_all();
    __syncwarp();
    // A: this lane's pixel
    const int64_t pix = base + lane;
    const double da = lane < P && pix < A.npix ? (A.d_alpha64 ? DAS[lane] : (double)reinterpret_cast<const float*>(DAS)[lane])
                                   : 0.0;
    const bool act = da != 0.0;  // shading.cpp:102: pixels with d_alpha == 0 contribute nothing
    const unsigned act_mask = __ballot_sync(0xffffffffu, act);
    const int64_t nslots = (A.npix - base < P ? A.npix - base : P) * K;
    int q = 0;
    if (act_mask) {
      const int rem = act ? (int)(pix % HW) : 0;
      const int i = rem / A.W, j = rem - i * A.W;
      PXY[2 * lane] = pixel_x(A.W, j);  // MR:357
      PXY[2 * lane + 1] = pixel_y(A.H, i);
      for (int t0 = 0; t0 < P * K; t0 += 32) {  // compacted in slot order
        const int t = t0 + lane;
        const int tp = t;
        const int64_t f = t < nslots ? STG[t] : -1;
        const bool occ = t < P * K && f >= 0 && f < A.F && ((act_mask >> (kK ? t / kK : (int)A.divK.div((uint32_t)t))) & 1u);
        if (t < P * K) {
          FID[tp] = occ ? (int32_t)f : -1;
          PR[tp] = -1.0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, occ);
        if (occ) Q[q + __popc(m & ((1u << lane) - 1u))] = (uint16_t)tp;
        q += __popc(m);
      }
    }
    __syncwarp();
    if (base + nwarps * P < A.npix) issue(base + nwarps * P);  // the staging buffers are free again
    if (!act_mask) continue;
    // B: envelope + prob per queued slot (next batch's face_verts prefetched)
    {
      double vn[9];
      int tn = lane < q ? Q[lane] : -1;
      int32_t fn = tn >= 0 ? FID[tn] : -1;
      if (fn >= 0) {
#pragma unroll
        for (int u = 0; u < 9; ++u) vn[u] = __ldg(A.fv + 9 * (int64_t)fn + u);
      }
      for (int q0 = 0; q0 < q; q0 += 32) {
        const int t = tn;
        double v[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) v[u] = vn[u];
        tn = q0 + 32 + lane < q ? Q[q0 + 32 + lane] : -1;
        fn = tn >= 0 ? FID[tn] : -1;
        if (fn >= 0) {
#pragma unroll
          for (int u = 0; u < 9; ++u) vn[u] = __ldg(A.fv + 9 * (int64_t)fn + u);
        }
        if (t >= 0) {
          const int pl = (kK ? t / kK : (int)A.divK.div((uint32_t)t));
          const V2 p{PXY[2 * pl], PXY[2 * pl + 1]};
          double dist, bt, sign;
          int be;
          V2 qq;
          silhouette_envelope(v, p, dist, be, bt, qq, sign);
          // sigmoid(-dist / sigma) (shading.cpp:9, 82): fp32 exp for the fp32 cotangent, fp64 for the fp64 one
          PR[t] = A.d_alpha64 ? fdiv(1.0, 1.0 + exp(dist * inv_sigma))
                              : fdiv(1.0, 1.0 + (double)expf((float)(dist * inv_sigma)));
          EX[t] = (qq.x - p.x) * (2.0 * sign);
          EY[t] = (qq.y - p.y) * (2.0 * sign);
          BT[t] = bt;
          BE[t] = be;
        }
      }
    }
    __syncwarp();
    // C: per pixel, d_dists (shading.cpp:115-117) = da * prod_{other occupied} (1 - prob) * (-prob (1 - prob) / sigma)
    if (act) {
      const int r = lane * KS;
      double suf = 1.0;
      for (int s = K - 1; s >= 0; --s) {
        CO[r + s] = suf;
        const double pr = PR[r + s];
        if (pr >= 0.0) suf *= 1.0 - pr;
      }
      double pre = 1.0;
      for (int s = 0; s < K; ++s) {
        const double pr = PR[r + s];
        if (pr >= 0.0) {
          CO[r + s] = da * (pre * CO[r + s]) * (-pr * (1.0 - pr) * inv_sigma);
          pre *= 1.0 - pr;
        }
      }
    }
    __syncwarp();
    // D: the frozen-edge envelope gradient (MR:46-69) per queued slot, summed per face across the warp
    for (int q0 = 0; q0 < q; q0 += 32) {
      const int t = q0 + lane < q ? Q[q0 + lane] : -1;
      int32_t fid = -1;
      double g[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (t >= 0) {
        fid = FID[t];
        const double d_out = CO[t];
        const double bt = BT[t];
        const int be = BE[t];
        const V2 gg{EX[t] * d_out, EY[t] * d_out};  // (qq - p) * (2 sign d_out): the same single rounding
        const V2 g_first = gg * (1.0 - bt), g_second = gg * bt;
        const int v1 = be == 2 ? 0 : be + 1;
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // vertex be gets g_first, the next one g_second (selects, no local array)
          g[2 * k] = be == k ? g_first.x : (v1 == k ? g_second.x : 0.0);
          g[2 * k + 1] = be == k ? g_first.y : (v1 == k ? g_second.y : 0.0);
        }
      }
      if (reduce_by_face<6>(fid, lane, g)) {
        double* out = A.grad + 9 * (int64_t)fid;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          atomicAdd(out + 3 * k, g[2 * k]);
          atomicAdd(out + 3 * k + 1, g[2 * k + 1]);
        }
      }
    }
    __syncwarp();
  }
}

cudaError_t launch_silhouette_backward(const SilBwdArgs& A, cudaStream_t st) {
  if (A.npix <= 0) return cudaSuccess;
  if (A.K <= kSilQMaxK) {  // (any K: chunks shrink to kSilQSlots / K pixels)
    const size_t smem = (size_t)kSilQWarps * silq_warp_bytes(A.K);
    auto kern = A.K == 8 ? k_silhouette_backward_q<8> : k_silhouette_backward_q<0>;
    SilBwdArgs B = A;
    B.divK = FastDivU32((uint32_t)A.K);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSilQWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (A.npix + (int64_t)kSilQWarps * silq_pixels(A.K) - 1) / ((int64_t)kSilQWarps * silq_pixels(A.K));
    if (blocks > need) blocks = need;
    kern<<<(unsigned)blocks, kSilQWarps * 32, smem, st>>>(B);
    return cudaGetLastError();
  }
  const bool store = A.K <= kSilStoreMaxK;
  const size_t per_warp = (size_t)A.K * 32 * (store ? 5 * sizeof(double) : 2 * sizeof(double)) +
                          (size_t)A.K * 16 * sizeof(double) * (store ? 2 : 1);  // + edge ids + the p2f block
  const int max_smem = 227 * 1024;
  if (per_warp > (size_t)max_smem) return cudaErrorInvalidConfiguration;
  const int warps = (int)std::min<size_t>(kSilThreads / 32, std::max<size_t>(1, (size_t)(96 * 1024) / per_warp));
  const size_t smem = per_warp * warps;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (A.npix + warps * 32 - 1) / (warps * 32);
    if (blocks > need) blocks = need;
    kern<<<(unsigned)blocks, warps * 32, smem, st>>>(A);
    return cudaGetLastError();
  };
  return store ? go(k_silhouette_backward<true>) : go(k_silhouette_backward<false>);
}

// ------------------------------------------------------------------------------------------------
// Fused softmax render backward: the reference's differentiable softmax render (grad.cpp:177-209) is
// rasterize_meshes -> interpolate_face_attributes(vertex colours) -> softmax_blend; its vjp chains
// softmax_blend_backward (shading.cpp:162-230) -> interpolate_face_attributes_backward (shading.cpp:35-73) ->
// rasterize_backward (MR:329-378). Here one lane per pixel walks its K slots: pass 1 re-evaluates each slot (fast
// divisions: values within tolerance) and keeps inverse depth, opacity and interpolated colour in shared memory;
// passes 2-3 form the softmax weights and the per-pixel mean term; pass 4 produces d_colors / d_dists / d_zbuf per
// slot (plus the zinv_max term on the argmax slot), d_bary_i = d_color . colour(v_i), the vertex-colour cotangent
// and the K3 per-slot chain, summed per face across the warp before the fp64 atomics.
// The argmax of zinv (shading.cpp:190-193, first strict maximum) is always the first occupied slot: slots are
// sorted ascending by (z, id) and zinv is non-increasing in z (clamping only creates equal values, and the first
// of equal values wins), so no exact depth is needed to reproduce the reference's choice under depth ties.

constexpr int kSoftThreads = 128;
constexpr int kSoftMaxK = 64;
constexpr int kSoftMaxGroupsPerCta = 32;

// clamped inverse depth (shading.cpp:136-137, 199) with the depth range's reciprocal precomputed (inv_zr)
__device__ __forceinline__ double blend_zinv_b(double z, const BlendArgs& bl, double inv_zr, bool& clamped) {
  clamped = z < bl.znear || z > bl.zfar;  // shading.cpp:199
  const double zc = z < bl.znear ? bl.znear : (bl.zfar < z ? bl.zfar : z);
  return (bl.zfar - zc) * inv_zr;
}

// one instantiation per (perspective_correct, clip_barycentric_coords), as K3: both the slot re-evaluation and the K3
// chain carry only their own branch (the kernel is instruction-cache bound)
// kK: K fixed at compile time (8, the headline K: constant shared-memory offsets), or 0 = read from A
template <int kPC, int kCL, int kK = 0>
__global__ void __launch_bounds__(kSoftThreads, 4) k_softmax_backward(SoftBwdArgs A, int gpc) {
  constexpr bool persp = kPC == 1, clip = kCL == 1;
  extern __shared__ double soft_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int K = kK ? kK : A.K;
  const size_t per_warp = (size_t)K * 32 * 6 + (size_t)K * 16;  // doubles
  // one base pointer and K * 32 live across the loops; the arrays' bases are formed at each use (separate pointer
  // registers had pushed ptxas into spilling one of them on the hot path)
  double* ZI = soft_smem + (size_t)wid * per_warp;  // [K][32] zinv (-1: empty slot; +2: clamped)
  const int K32 = K * 32;
#define PR (ZI + K32)                                    // [K][32] prob
#define WT (ZI + 2 * K32)                                // [K][32] softmax weight
#define C0 (ZI + 3 * K32)                                // [K][32] interpolated colour
#define C1 (ZI + 4 * K32)
#define C2 (ZI + 5 * K32)
#define FID (reinterpret_cast<int32_t*>(ZI + 6 * K32))  // [32][K] the warp's pix_to_face block
  BwdArgs<double> BA;  // the K3 per-slot chain's flags
  BA.persp = A.persp;
  BA.clip = A.clip;
  __shared__ int next_group;
  if (threadIdx.x == 0) next_group = blockDim.x >> 5;  // group w is warp w's first
  __syncthreads();
  const int64_t HW = (int64_t)A.H * A.W;
  // the blend's divisions by sigma, gamma, the depth range and the per-pixel weight sum become products with
  // reciprocals (values compared within tolerance, never selected on: <= 2 ulp from the quotients; C4 10.7 -> 8.8 ms)
  // (the host's reciprocals, BlendArgs::inv_*: kernel-parameter operands, no registers held across the loop)
#define inv_sigma (A.blend.inv_sigma)
#define inv_gamma (A.blend.inv_gamma)
#define inv_zr (A.blend.inv_zr)
#define SDIV_SIGMA(x) ((x) * inv_sigma)
#define SDIV_GAMMA(x) ((x) * inv_gamma)
  // the CTA's gpc consecutive 32-pixel groups are taken by its warps from a shared counter (many CTAs, balanced by
  // the block scheduler, instead of a persistent grid whose warps finish unevenly: C4 8.11 -> 6.5-6.8 ms)
  const int g0 = (int)blockIdx.x * gpc;  // group indices fit 32 bits (the launcher caps the grid at INT32_MAX)
  int kg = wid;
  while (kg < gpc && (int64_t)(g0 + kg) * 32 < A.npix) {
    const int64_t base = (int64_t)(g0 + kg) * 32;
    const int64_t pix = base + lane;
    double dimg[3] = {0.0, 0.0, 0.0};
    if (pix < A.npix) {
      dimg[0] = (double)A.d_image[3 * pix];
      dimg[1] = (double)A.d_image[3 * pix + 1];
      dimg[2] = (double)A.d_image[3 * pix + 2];
    }
    {
      const int64_t n = (A.npix - base < 32 ? A.npix - base : 32) * K;
      const int64_t* src = A.p2f + base * K;
      for (int t = lane; t < 32 * K; t += 32) {
        const int64_t f = t < n ? __ldcs(src + t) : -1;
        FID[t] = (f >= 0 && f < A.F) ? (int32_t)f : -1;
      }
      __syncwarp();
    }
    const int32_t* row = FID + lane * K;
    const int rem = pix < A.npix ? (int)(pix % HW) : 0;
    const int i = rem / A.W, j = rem - (rem / A.W) * A.W;
    const V2 p{pixel_x(A.W, j), pixel_y(A.H, i)};
    // pass 1: exact slot evaluation, zinv_max / argmax (shading.cpp:185-197)
    double zinv_max = -1.0;
    int argmax = -1;
    bool any = false;
#pragma unroll 1
    for (int s = 0; s < K; ++s) {
      const int32_t f = pix < A.npix ? row[s] : -1;
      double zi = -1.0;
      if (f >= 0) {
        any = true;
        double v[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) v[t] = __ldg(A.fv + 9 * (int64_t)f + t);
        const FaceGeom g = make_face_geom(v);
        PixelFaceResult r;
        eval_pixel_face<true, false>(p, g, A.blur, A.znear, persp, clip, r);
        bool clamped;
        zi = blend_zinv_b(r.z, A.blend, inv_zr, clamped);
        if (argmax < 0) {  // the first occupied slot (see above)
          zinv_max = zi;
          argmax = s;
        }
        double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 3; ++q) {  // interpolate_face_attributes (shading.cpp:21-29)
          const double* a = A.blend.vert_colors + 3 * A.blend.faces[3 * (int64_t)f + q];
          c[0] += r.bary[q] * __ldg(a);
          c[1] += r.bary[q] * __ldg(a + 1);
          c[2] += r.bary[q] * __ldg(a + 2);
        }
        C0[s * 32 + lane] = c[0];
        C1[s * 32 + lane] = c[1];
        C2[s * 32 + lane] = c[2];
        PR[s * 32 + lane] = fdiv(1.0, 1.0 + exp(SDIV_SIGMA(r.dist)));  // sigmoid(-dists / sigma)
        if (clamped) zi += 2.0;
      }
      ZI[s * 32 + lane] = zi;
    }
    // pass 2: weights and their sum (shading.cpp:202-209)
    double wsum = 0.0;
    for (int s = 0; s < K; ++s) {
      double zi = ZI[s * 32 + lane];
      if (zi < -0.5) continue;
      if (zi > 1.5) zi -= 2.0;
      const double w = PR[s * 32 + lane] * exp(SDIV_GAMMA(zi - zinv_max));
      WT[s * 32 + lane] = w;
      wsum += w;
    }
    // pass 3: the mean term (shading.cpp:218-222; identical for every slot, computed once in the same order)
    const double inv_wsum = fdiv(1.0, wsum);
#define SDIV_WSUM(x) ((x) * inv_wsum)
    double mean_term = 0.0;
    for (int s = 0; s < K; ++s) {
      if (ZI[s * 32 + lane] < -0.5) continue;
      const double dc = dimg[0] * C0[s * 32 + lane] + dimg[1] * C1[s * 32 + lane] + dimg[2] * C2[s * 32 + lane];
      mean_term += dc * SDIV_WSUM(WT[s * 32 + lane]);
    }
    // d_zinv_max (shading.cpp:228) before the per-slot pass that adds it to the argmax slot
    double d_zinv_max = 0.0;
    for (int s = 0; s < K; ++s) {
      if (ZI[s * 32 + lane] < -0.5) continue;
      const double w = WT[s * 32 + lane];
      const double d_what = dimg[0] * C0[s * 32 + lane] + dimg[1] * C1[s * 32 + lane] + dimg[2] * C2[s * 32 + lane];
      const double d_w = SDIV_WSUM(d_what - mean_term);
      d_zinv_max += SDIV_GAMMA(-d_w * w);
    }
    // pass 4: per-slot cotangents -> colours, barycentrics, the K3 chain
#pragma unroll 1
    for (int s = 0; s < K; ++s) {
      const double zis = (pix < A.npix && any) ? ZI[s * 32 + lane] : -1.0;
      int32_t fid = -1;
      double g[9], gc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) g[k] = gc[k] = 0.0;
      if (zis >= -0.5) {
        fid = row[s];
        const bool clamped = zis > 1.5;
        const double w = WT[s * 32 + lane], pr = PR[s * 32 + lane];
        const double c[3] = {C0[s * 32 + lane], C1[s * 32 + lane], C2[s * 32 + lane]};
        const double what = SDIV_WSUM(w);
        const double d_col[3] = {dimg[0] * what, dimg[1] * what, dimg[2] * what};  // g.d_colors = dimg * what
        const double d_what = dimg[0] * c[0] + dimg[1] * c[1] + dimg[2] * c[2];
        const double d_w = SDIV_WSUM(d_what - mean_term);
        const double d_prob = fdiv(d_w * w, pr);
        const double d_zinv = SDIV_GAMMA(d_w * w);
        const double d_dists = d_prob * SDIV_SIGMA(-pr * (1.0 - pr));
        double d_zbuf = clamped ? 0.0 : d_zinv * -inv_zr;
        if (s == argmax && !clamped) d_zbuf += d_zinv_max * -inv_zr;
        // interpolate_face_attributes_backward (shading.cpp:46-72): d_bary_i = d_col . a_i, d_attr_i += w_i d_col
        SlotIn<double> in;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double* a = A.blend.vert_colors + 3 * A.blend.faces[3 * (int64_t)fid + q];
          in.db[q] = d_col[0] * __ldg(a) + d_col[1] * __ldg(a + 1) + d_col[2] * __ldg(a + 2);
          in.w[q] = 0.0;
        }
        in.dz = d_zbuf;
        in.dd = d_dists;
#pragma unroll
        for (int t = 0; t < 9; ++t) in.v[t] = __ldg(A.fv + 9 * (int64_t)fid + t);
        double wh[3];
        slot_backward<double, true, kPC, kCL>(BA, p, fid, in, g, wh);  // the slot's clamped barycentrics come back in wh
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          gc[3 * q + 0] = wh[q] * d_col[0];
          gc[3 * q + 1] = wh[q] * d_col[1];
          gc[3 * q + 2] = wh[q] * d_col[2];
        }
      }
      // one reduction over 18 values: the face_verts cotangent and the face's vertex-colour cotangents
      double gg[18];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        gg[k] = g[k];
        gg[9 + k] = gc[k];
      }
      if (reduce_by_face<18>(fid, lane, gg)) {
        // the face's vertex ids (L1) before the face_verts atomics, so those cover the load's latency
        int64_t vi[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) vi[q] = __ldg(A.blend.faces + 3 * (int64_t)fid + q);
        double* out = A.grad + 9 * (int64_t)fid;
#pragma unroll
        for (int k = 0; k < 9; ++k)
          if (gg[k] != 0.0) atomicAdd(out + k, gg[k]);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double* oc = A.grad_colors + 3 * vi[q];
          for (int d = 0; d < 3; ++d)
            if (gg[9 + 3 * q + d] != 0.0) atomicAdd(oc + d, gg[9 + 3 * q + d]);
        }
      }
    }
    int kn = 0;
    if (lane == 0) kn = atomicAdd(&next_group, 1);
    kg = __shfl_sync(0xffffffffu, kn, 0);
  }
}
#undef PR
#undef WT
#undef C0
#undef C1
#undef C2
#undef FID
#undef inv_sigma
#undef inv_gamma
#undef inv_zr
#undef SDIV_SIGMA
#undef SDIV_GAMMA
#undef SDIV_WSUM

// Slot-compacted variant: a warp takes P = min(32, kSoftQSlots / K) consecutive pixels; their occupied slots are queued
// and the two geometry-heavy passes run lane-per-slot, 32 occupied slots per step:
//   B  per slot: exact-sequence re-evaluation (fast divisions), inverse depth, opacity, interpolated colour
//   C  per pixel (lane < P): zinv_max (the first occupied slot, see above), weights, the mean term, d_zinv_max,
//      then per slot what = w / wsum, d_dists and d_zbuf (same operation order as the per-pixel kernel)
//   D  per slot: d_bary from the vertex colours, the K3 chain, the colour cotangent, one 18-value reduce-by-face
// at most 320 slots per chunk (C5, K=50: 6 pixels 8.96 ms vs 10 pixels 9.46, 5 pixels 9.29, 7 pixels 9.11)
constexpr int kSoftQSlots = 320;

__host__ __device__ __forceinline__ int softq_pixels(int K) { return K >= kSoftQSlots ? 1 : min(32, kSoftQSlots / K); }
__host__ __device__ __forceinline__ size_t softq_warp_bytes(int K) {
  const size_t n = (size_t)softq_pixels(K) * K;
  return n * (6 * sizeof(double) + sizeof(int32_t) + sizeof(uint16_t)) + 32 * 5 * sizeof(double) + 16;
}

template <int kPC, int kCL>
__global__ void __launch_bounds__(32) k_softmax_backward_q(SoftBwdArgs A) {
  constexpr bool persp = kPC == 1, clip = kCL == 1;
  // as k_softmax_backward: products with reciprocals instead of the blend's divisions (tolerance values)
  const double inv_sigma = 1.0 / A.blend.sigma, inv_gamma = 1.0 / A.blend.gamma,
               inv_zr = 1.0 / (A.blend.zfar - A.blend.znear);
  extern __shared__ double softq_smem[];
  const int lane = threadIdx.x & 31;
  const int K = A.K;
  const int P = softq_pixels(K);
  const int KS = K;  // per-pixel row stride (K + 1, conflict-free for the lane-per-pixel pass, measured slower)
  const int n = P * KS;
  double* ZI = softq_smem;  // [n] zinv (-1: empty; +2: clamped), then d_zbuf
  double* PR = ZI + n;      // [n] prob, then d_dists
  double* WT = PR + n;      // [n] weight, then what = w / wsum
  double* C0 = WT + n;      // [n] interpolated colour
  double* C1 = C0 + n;
  double* C2 = C1 + n;
  double* PXY = C2 + n;     // [32][2] pixel centres
  double* DIM = PXY + 64;   // [32][3] d_image
  int32_t* FID = reinterpret_cast<int32_t*>(DIM + 96);  // [n]
  uint16_t* Q = reinterpret_cast<uint16_t*>(FID + n);   // [n]
  BwdArgs<double> BA;
  BA.persp = A.persp;
  BA.clip = A.clip;
  const int64_t HW = (int64_t)A.H * A.W;
  for (int64_t base = (int64_t)blockIdx.x * P; base < A.npix; base += (int64_t)gridDim.x * P) {
    const int np = (int)(A.npix - base < P ? A.npix - base : P);
    if (lane < np) {
      const int64_t pix = base + lane;
      const int rem = (int)(pix % HW);
      const int i = rem / A.W, j = rem - i * A.W;
      PXY[2 * lane] = pixel_x(A.W, j);  // MR:357
      PXY[2 * lane + 1] = pixel_y(A.H, i);
      DIM[3 * lane] = (double)A.d_image[3 * pix];
      DIM[3 * lane + 1] = (double)A.d_image[3 * pix + 1];
      DIM[3 * lane + 2] = (double)A.d_image[3 * pix + 2];
    }
    // A: pix_to_face block -> queue of occupied slots (slot order; a (rank, pixel) order that groups shared
    // faces for reduce_by_face measured slower: C4 15.1 -> 16.8 ms)
    const int ns = np * K;
    const int64_t* src = A.p2f + base * K;
    int q = 0;
    for (int t0 = 0; t0 < P * K; t0 += 32) {
      const int t = t0 + lane;
      const int tp = t;
      const int64_t f = t < ns ? __ldcs(src + t) : -1;
      const bool occ = f >= 0 && f < A.F;
      if (t < P * K) {
        FID[tp] = occ ? (int32_t)f : -1;
        ZI[tp] = -1.0;
      }
      const unsigned m = __ballot_sync(0xffffffffu, occ);
      if (occ) Q[q + __popc(m & ((1u << lane) - 1u))] = (uint16_t)tp;
      q += __popc(m);
    }
    __syncwarp();
    // B: per occupied slot
    {
      double vn[9];
      int tn = lane < q ? Q[lane] : -1;
      int32_t fn = tn >= 0 ? FID[tn] : -1;
      if (fn >= 0) {
#pragma unroll
        for (int u = 0; u < 9; ++u) vn[u] = __ldg(A.fv + 9 * (int64_t)fn + u);
      }
      for (int q0 = 0; q0 < q; q0 += 32) {
        const int t = tn;
        const int32_t f = fn;
        double v[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) v[u] = vn[u];
        tn = q0 + 32 + lane < q ? Q[q0 + 32 + lane] : -1;
        fn = tn >= 0 ? FID[tn] : -1;
        if (fn >= 0) {
#pragma unroll
          for (int u = 0; u < 9; ++u) vn[u] = __ldg(A.fv + 9 * (int64_t)fn + u);
        }
        if (t >= 0) {
          const int pl = (int)A.divK.div((uint32_t)t);
          const V2 p{PXY[2 * pl], PXY[2 * pl + 1]};
          const FaceGeom g = make_face_geom(v);
          PixelFaceResult r;
          eval_pixel_face<true, false>(p, g, A.blur, A.znear, persp, clip, r);
          bool clamped;
          double zi = blend_zinv_b(r.z, A.blend, inv_zr, clamped);
          double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
          for (int qq = 0; qq < 3; ++qq) {  // interpolate_face_attributes (shading.cpp:21-29)
            const double* a = A.blend.vert_colors + 3 * A.blend.faces[3 * (int64_t)f + qq];
            c[0] += r.bary[qq] * __ldg(a);
            c[1] += r.bary[qq] * __ldg(a + 1);
            c[2] += r.bary[qq] * __ldg(a + 2);
          }
          C0[t] = c[0];
          C1[t] = c[1];
          C2[t] = c[2];
          PR[t] = fdiv(1.0, 1.0 + exp(r.dist * inv_sigma));  // sigmoid(-dists / sigma)
          if (clamped) zi += 2.0;
          ZI[t] = zi;
        }
      }
    }
    __syncwarp();
    // C: per pixel (shading.cpp:185-228)
    if (lane < np) {
      const int r0 = lane * KS;
      const double dimg[3] = {DIM[3 * lane], DIM[3 * lane + 1], DIM[3 * lane + 2]};
      double zinv_max = -1.0;
      int argmax = -1;
      for (int s = 0; s < K; ++s) {
        double zi = ZI[r0 + s];
        if (zi < -0.5) continue;
        if (zi > 1.5) zi -= 2.0;
        if (argmax < 0) {
          zinv_max = zi;
          argmax = s;
        }
      }
      double wsum = 0.0;
      for (int s = 0; s < K; ++s) {
        double zi = ZI[r0 + s];
        if (zi < -0.5) continue;
        if (zi > 1.5) zi -= 2.0;
        const double w = PR[r0 + s] * exp((zi - zinv_max) * inv_gamma);
        WT[r0 + s] = w;
        wsum += w;
      }
      const double inv_wsum = fdiv(1.0, wsum);
      double mean_term = 0.0;
      for (int s = 0; s < K; ++s) {
        if (ZI[r0 + s] < -0.5) continue;
        const double dc = dimg[0] * C0[r0 + s] + dimg[1] * C1[r0 + s] + dimg[2] * C2[r0 + s];
        mean_term += dc * (WT[r0 + s] * inv_wsum);
      }
      double d_zinv_max = 0.0;
      for (int s = 0; s < K; ++s) {
        if (ZI[r0 + s] < -0.5) continue;
        const double w = WT[r0 + s];
        const double d_what = dimg[0] * C0[r0 + s] + dimg[1] * C1[r0 + s] + dimg[2] * C2[r0 + s];
        const double d_w = (d_what - mean_term) * inv_wsum;
        d_zinv_max += -d_w * w * inv_gamma;
      }
      for (int s = 0; s < K; ++s) {
        const double zis = ZI[r0 + s];
        if (zis < -0.5) continue;
        const bool clamped = zis > 1.5;
        const double w = WT[r0 + s], pr = PR[r0 + s];
        const double what = w * inv_wsum;
        const double d_what = dimg[0] * C0[r0 + s] + dimg[1] * C1[r0 + s] + dimg[2] * C2[r0 + s];
        const double d_w = (d_what - mean_term) * inv_wsum;
        const double d_prob = fdiv(d_w * w, pr);
        const double d_zinv = d_w * w * inv_gamma;
        const double d_dists = d_prob * (-pr * (1.0 - pr) * inv_sigma);
        double d_zbuf = clamped ? 0.0 : d_zinv * -inv_zr;
        if (s == argmax && !clamped) d_zbuf += d_zinv_max * -inv_zr;
        WT[r0 + s] = what;
        PR[r0 + s] = d_dists;
        ZI[r0 + s] = d_zbuf;
      }
    }
    __syncwarp();
    // D: per occupied slot
    for (int q0 = 0; q0 < q; q0 += 32) {
      const int t = q0 + lane < q ? Q[q0 + lane] : -1;
      int32_t fid = -1;
      double gg[18];
#pragma unroll
      for (int k = 0; k < 18; ++k) gg[k] = 0.0;
      if (t >= 0) {
        fid = FID[t];
        const int pl = (int)A.divK.div((uint32_t)t);
        const V2 p{PXY[2 * pl], PXY[2 * pl + 1]};
        const double what = WT[t];
        const double d_col[3] = {DIM[3 * pl] * what, DIM[3 * pl + 1] * what, DIM[3 * pl + 2] * what};
        SlotIn<double> in;
#pragma unroll
        for (int qq = 0; qq < 3; ++qq) {  // interpolate_face_attributes_backward (shading.cpp:46-72)
          const double* a = A.blend.vert_colors + 3 * A.blend.faces[3 * (int64_t)fid + qq];
          in.db[qq] = d_col[0] * __ldg(a) + d_col[1] * __ldg(a + 1) + d_col[2] * __ldg(a + 2);
          in.w[qq] = 0.0;
        }
        in.dz = ZI[t];
        in.dd = PR[t];
#pragma unroll
        for (int u = 0; u < 9; ++u) in.v[u] = __ldg(A.fv + 9 * (int64_t)fid + u);
        double g[9], wh[3];
        slot_backward<double, true, kPC, kCL>(BA, p, fid, in, g, wh);
#pragma unroll
        for (int k = 0; k < 9; ++k) gg[k] = g[k];
#pragma unroll
        for (int qq = 0; qq < 3; ++qq) {
          gg[9 + 3 * qq + 0] = wh[qq] * d_col[0];
          gg[9 + 3 * qq + 1] = wh[qq] * d_col[1];
          gg[9 + 3 * qq + 2] = wh[qq] * d_col[2];
        }
      }
      if (reduce_by_face<18>(fid, lane, gg)) {
        // the face's vertex ids (L1) before the face_verts atomics, so those cover the load's latency
        int64_t vi[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) vi[q] = __ldg(A.blend.faces + 3 * (int64_t)fid + q);
        double* out = A.grad + 9 * (int64_t)fid;
#pragma unroll
        for (int k = 0; k < 9; ++k)
          if (gg[k] != 0.0) atomicAdd(out + k, gg[k]);
#pragma unroll
        for (int qq = 0; qq < 3; ++qq) {
          double* oc = A.grad_colors + 3 * vi[qq];
          for (int d = 0; d < 3; ++d)
            if (gg[9 + 3 * qq + d] != 0.0) atomicAdd(oc + d, gg[9 + 3 * qq + d]);
        }
      }
    }
    __syncwarp();
  }
}

template <int kPC, int kCL>
static cudaError_t launch_softmax_backward_t(const SoftBwdArgs& A, cudaStream_t st) {
  // measured (C4 K=8 / C5 K=50): per-pixel kernel 10.9 / 39.1 ms, slot-compacted 15.1 / 16.1 ms — the
  // compaction pays once a pixel's K slots are unevenly filled (large K)
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // (a two-kernel form for K <= 16, coefficients through an [S][3] scratch, measured 11.6 vs 10.9 ms per-pixel)
  if (A.K > 16) {
    auto kern = k_softmax_backward_q<kPC, kCL>;
    const size_t smem = softq_warp_bytes(A.K);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t blocks = (int64_t)sms * per_sm;
    const int P = softq_pixels(A.K);
    const int64_t need = (A.npix + P - 1) / P;
    if (blocks > need) blocks = need;
    SoftBwdArgs B = A;
    B.divK = FastDivU32((uint32_t)A.K);
    kern<<<(unsigned)blocks, 32, smem, st>>>(B);
    return cudaGetLastError();
  }
  auto kern = A.K == 8 ? k_softmax_backward<kPC, kCL, 8> : k_softmax_backward<kPC, kCL>;
  const size_t per_warp = ((size_t)A.K * 32 * 6 + (size_t)A.K * 16) * sizeof(double);
  const int warps = (int)std::min<size_t>(kSoftThreads / 32, std::max<size_t>(1, (size_t)(96 * 1024) / per_warp));
  const size_t smem = per_warp * warps;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // groups per CTA: up to kSoftMaxGroupsPerCta, fewer when the image set is small (at least ~4 waves of CTAs; one
  // group per warp at the floor) — C2 with 32 per CTA filled only 128 of 148 SMs
  const int64_t groups = (A.npix + 31) / 32;
  const int64_t gpc = std::max<int64_t>(warps, std::min<int64_t>(kSoftMaxGroupsPerCta, groups / (4 * (int64_t)sms * per_sm)));
  const int64_t blocks = std::min<int64_t>((groups + gpc - 1) / gpc, INT32_MAX);
  kern<<<(unsigned)blocks, warps * 32, smem, st>>>(A, (int)gpc);
  return cudaGetLastError();
}

cudaError_t launch_softmax_backward(const SoftBwdArgs& A, cudaStream_t st) {
  if (A.npix <= 0) return cudaSuccess;
  if (A.K > kSoftMaxK) return cudaErrorInvalidConfiguration;
  if (A.persp) return A.clip ? launch_softmax_backward_t<1, 1>(A, st) : launch_softmax_backward_t<1, 0>(A, st);
  return A.clip ? launch_softmax_backward_t<0, 1>(A, st) : launch_softmax_backward_t<0, 0>(A, st);
}

template <typename InT>
static cudaError_t launch_backward_t(const BwdArgs<InT>& A, cudaStream_t st) {
  if (A.S <= 0) return cudaSuccess;
  // many CTAs of up to kBwdMaxChunksPerCta chunks instead of one persistent wave: the block scheduler then balances the
  // uneven per-chunk work (occupied-slot density varies across the image); a single wave measured 10.8 of 16
  // achievable warps per SM on C4
  // chunks per CTA: 32 for the large configs (C4: 16 per CTA 2.28 ms, 8 2.58 vs 2.25), fewer once that leaves less
  // than ~2 waves of CTAs (C2, 2,048 chunks: 32 per CTA filled 64 of 148 SMs, 0.155 ms; 8 per CTA 0.050)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nchunks = (A.S + kBwdChunk - 1) / kBwdChunk;
  BwdArgs<InT> B = A;
  B.cpc = (int)std::max<int64_t>(kBwdThreads / 32,  // at least one chunk per warp
                                 std::min<int64_t>(kBwdMaxChunksPerCta, nchunks / (2 * (int64_t)sms * kBwdMinBlocks)));
  const int64_t blocks = std::min<int64_t>((nchunks + B.cpc - 1) / B.cpc, INT32_MAX);
  // one instantiation per (perspective_correct, clip_barycentric_coords)
  auto go = [&](auto kern) {
    kern<<<(unsigned)blocks, kBwdThreads, 0, st>>>(B);
    return cudaGetLastError();
  };
  if (A.persp) return A.clip ? go(k_backward<InT, 1, 1>) : go(k_backward<InT, 1, 0>);
  return A.clip ? go(k_backward<InT, 0, 1>) : go(k_backward<InT, 0, 0>);
}

cudaError_t launch_backward(const BwdArgs<float>& A, cudaStream_t st) { return launch_backward_t(A, st); }
cudaError_t launch_backward(const BwdArgs<double>& A, cudaStream_t st) { return launch_backward_t(A, st); }

}  // namespace drb
