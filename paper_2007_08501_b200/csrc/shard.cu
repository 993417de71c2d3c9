// Mesh sharding plan and the fragment gather's operation list (host code).
//
// Meshes are the shard unit: the reference processes them one after another and nothing crosses meshes
// (mesh_raster.cpp:240-283 forward, 380-401 backward per face range). A rank rasterizes its meshes with their
// GLOBAL ranges of the packed batch (mesh_to_face_first_idx / num_faces_per_mesh of those meshes), so pix_to_face
// holds global packed face ids and the backward writes only the rank's own rows of grad_face_verts — no id
// translation and no collective on the data path. The optional gather to one rank is a list of point-to-point
// transfers computed here identically on every rank (include/dr_shard.h); libdr_shard_b200.so executes it with
// NCCL, the CPU tests with torch.distributed over gloo.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <queue>
#include <vector>

#include "../../include/dr_shard.h"

extern "C" int dr_set_error(int status, const char* msg);  // capi.cu: thread-local dr_last_error()

namespace {

int err(int status, const char* msg) { return dr_set_error(status, msg); }

}  // namespace

extern "C" int dr_shard_plan_lpt(const int64_t* costs, int64_t N, int32_t nranks, int32_t* owner,
                                 int32_t* local_index) {
  if (N < 0 || nranks < 1) return err(DR_ERR_SHAPE, "dr_shard_plan_lpt: N < 0 or nranks < 1");
  if (N > 0 && (!costs || !owner || !local_index)) return err(DR_ERR_USAGE, "dr_shard_plan_lpt: null pointer");
  // longest processing time first: items by decreasing cost (ties: lower index), each to the least-loaded rank
  // (ties: lower rank)
  std::vector<int64_t> order((size_t)N);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return costs[a] > costs[b]; });
  using Slot = std::pair<double, int32_t>;  // (load, rank)
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int32_t r = 0; r < nranks; ++r) heap.push({0.0, r});
  for (int64_t i : order) {
    if (costs[i] < 0) return err(DR_ERR_RANGE, "dr_shard_plan_lpt: negative cost");
    Slot s = heap.top();
    heap.pop();
    owner[i] = s.second;
    heap.push({s.first + (double)costs[i], s.second});
  }
  // local index = position of the mesh in its owner's ascending mesh list (the order of the rank's outputs)
  std::vector<int32_t> next((size_t)nranks, 0);
  for (int64_t m = 0; m < N; ++m) local_index[m] = next[(size_t)owner[m]]++;
  return DR_OK;
}

extern "C" int dr_shard_gather_ops(int64_t N, const int32_t* owner, const int32_t* local_index,
                                   const int64_t* mesh_first, const int64_t* mesh_num, int64_t slots_per_mesh,
                                   int32_t payload_bytes, int32_t with_grad, int32_t nranks, int32_t rank,
                                   int32_t root, int32_t local_lo, int32_t local_hi, dr_shard_op* ops, int64_t cap,
                                   int64_t* n_ops) {
  if (!n_ops) return err(DR_ERR_USAGE, "dr_shard_gather_ops: n_ops is null");
  *n_ops = 0;
  if (N < 0 || slots_per_mesh < 0) return err(DR_ERR_SHAPE, "dr_shard_gather_ops: negative sizes");
  if (payload_bytes != 4 && payload_bytes != 8)
    return err(DR_ERR_RANGE, "dr_shard_gather_ops: payload_bytes must be 4 (fp32) or 8 (fp64)");
  if (nranks < 1 || rank < 0 || rank >= nranks || root < 0 || root >= nranks)
    return err(DR_ERR_RANGE, "dr_shard_gather_ops: rank / root outside [0, nranks)");
  if (N > 0 && (!owner || !local_index || (with_grad && (!mesh_first || !mesh_num))))
    return err(DR_ERR_USAGE, "dr_shard_gather_ops: null plan pointer");
  for (int64_t m = 0; m < N; ++m) {
    if (owner[m] < 0 || owner[m] >= nranks) return err(DR_ERR_INDEX, "dr_shard_gather_ops: owner outside ranks");
    if (local_index[m] < 0) return err(DR_ERR_INDEX, "dr_shard_gather_ops: negative local index");
    if (with_grad && (mesh_first[m] < 0 || mesh_num[m] < 0))
      return err(DR_ERR_INDEX, "dr_shard_gather_ops: negative mesh range");
  }
  // per buffer: element bytes of one slot (pix_to_face int64; zbuf / dists one payload value; bary three)
  const int64_t eb[4] = {8, payload_bytes, 3 * (int64_t)payload_bytes, payload_bytes};
  int64_t n = 0;
  auto emit = [&](int32_t kind, int32_t peer, int32_t buf, int64_t m, int64_t src, int64_t dst, int64_t bytes) {
    if (bytes <= 0) return;
    if (ops && n < cap) {
      ops[n].kind = kind;
      ops[n].peer = peer;
      ops[n].buffer = buf;
      ops[n].mesh = (int32_t)m;
      ops[n].src_offset = src;
      ops[n].dst_offset = dst;
      ops[n].bytes = bytes;
    }
    ++n;
  };
  // meshes in ascending global order, buffers in a fixed order: every (sender, root) pair enumerates its
  // transfers in the same sequence on both sides, which is how point-to-point sends and receives are matched
  for (int64_t m = 0; m < N; ++m) {
    const int32_t o = owner[m], li = local_index[m];
    if (li < local_lo || li >= local_hi) continue;
    const bool mine = o == rank;
    const int32_t kind = o == root ? (rank == root ? DR_SHARD_COPY : -1)
                                   : (mine ? DR_SHARD_SEND : (rank == root ? DR_SHARD_RECV : -1));
    if (kind < 0) continue;
    const int32_t peer = kind == DR_SHARD_SEND ? root : o;
    for (int b = 0; b < 4; ++b) {
      const int64_t bytes = slots_per_mesh * eb[b];
      emit(kind, peer, b, m, (int64_t)li * bytes, m * bytes, bytes);
    }
    if (with_grad) {  // grad_face_verts rows of the mesh: the same rows of [F,3,3] on every rank
      const int64_t off = mesh_first[m] * 72, bytes = mesh_num[m] * 72;
      emit(kind, peer, DR_BUF_GRAD, m, off, off, bytes);
    }
  }
  *n_ops = n;
  if (ops && n > cap) return err(DR_ERR_OOM, "dr_shard_gather_ops: op buffer too small");
  return DR_OK;
}
