// libdr_shard_b200.so: the fragment gather of a mesh-sharded batch executed with NCCL (include/dr_shard.h).
//
// The op list comes from dr_shard_gather_ops (libdr_raster_b200.so, identical on every rank); here it becomes one
// NCCL group of ncclSend / ncclRecv (NVLink / NVSwitch point-to-point, all of a call's transfers in flight at
// once) plus cudaMemcpyAsync device copies for the root's own meshes, all on the caller's stream. Kept out of
// libdr_raster_b200.so so the rasterizer itself does not depend on NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dr_shard.h"

struct dr_shard_comm {
  ncclComm_t comm = nullptr;
  int32_t nranks = 0, rank = 0;
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int nccl_fail(ncclResult_t r, const char* where) {
  return fail(DR_ERR_CUDA, "NCCL error in %s: %s", where, ncclGetErrorString(r));
}

char* at(void* base, int64_t off) { return static_cast<char*>(base) + off; }

void* buffer(const dr_shard_buffers* b, int32_t id) {
  switch (id) {
    case DR_BUF_P2F: return b->pix_to_face;
    case DR_BUF_ZBUF: return b->zbuf;
    case DR_BUF_BARY: return b->bary;
    case DR_BUF_DISTS: return b->dists;
    default: return b->grad_face_verts;
  }
}

}  // namespace

extern "C" {

const char* dr_shard_last_error(void) { return g_err.c_str(); }

int dr_shard_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  if (!id) return fail(DR_ERR_USAGE, "dr_shard_unique_id: null pointer");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return DR_OK;
}

int dr_shard_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], dr_shard_comm_t* comm) {
  if (!id || !comm) return fail(DR_ERR_USAGE, "dr_shard_comm_init: null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(DR_ERR_RANGE, "dr_shard_comm_init: bad rank");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  auto* c = new dr_shard_comm;
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  *comm = c;
  return DR_OK;
}

int dr_shard_comm_destroy(dr_shard_comm_t comm) {
  if (!comm) return DR_OK;
  ncclResult_t r = ncclCommDestroy(comm->comm);
  delete comm;
  return r == ncclSuccess ? DR_OK : nccl_fail(r, "ncclCommDestroy");
}

int dr_shard_gather(dr_shard_comm_t comm, int32_t root, int64_t N, const int32_t* owner, const int32_t* local_index,
                    const int64_t* mesh_first, const int64_t* mesh_num, int64_t slots_per_mesh,
                    int32_t payload_bytes, int32_t with_grad, int32_t local_lo, int32_t local_hi,
                    const dr_shard_buffers* local, const dr_shard_buffers* global, dr_stream_t stream) {
  if (!comm || !local) return fail(DR_ERR_USAGE, "dr_shard_gather: null comm / buffers");
  if (comm->rank == root && !global) return fail(DR_ERR_USAGE, "dr_shard_gather: the root needs global buffers");
  int64_t n = 0;
  int rc = dr_shard_gather_ops(N, owner, local_index, mesh_first, mesh_num, slots_per_mesh, payload_bytes, with_grad,
                               comm->nranks, comm->rank, root, local_lo, local_hi, nullptr, 0, &n);
  if (rc) return fail(rc, "dr_shard_gather: %s", dr_last_error());
  std::vector<dr_shard_op> ops((size_t)n);
  rc = dr_shard_gather_ops(N, owner, local_index, mesh_first, mesh_num, slots_per_mesh, payload_bytes, with_grad,
                           comm->nranks, comm->rank, root, local_lo, local_hi, ops.data(), n, &n);
  if (rc) return fail(rc, "dr_shard_gather: %s", dr_last_error());
  for (const dr_shard_op& op : ops) {
    void* src = buffer(local, op.buffer);
    void* dst = op.kind == DR_SHARD_SEND ? nullptr : buffer(global, op.buffer);
    if ((op.kind != DR_SHARD_RECV && !src) || (op.kind != DR_SHARD_SEND && !dst))
      return fail(DR_ERR_USAGE, "dr_shard_gather: buffer %d is null", op.buffer);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // the root's own meshes: device copies, enqueued before the group (they do not depend on the transfers)
  for (const dr_shard_op& op : ops) {
    if (op.kind != DR_SHARD_COPY) continue;
    char* s = at(buffer(local, op.buffer), op.src_offset);
    char* d = at(buffer(global, op.buffer), op.dst_offset);
    if (s == d) continue;
    cudaError_t e = cudaMemcpyAsync(d, s, (size_t)op.bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return fail(DR_ERR_CUDA, "dr_shard_gather copy: %s", cudaGetErrorString(e));
  }
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (const dr_shard_op& op : ops) {
    if (op.kind == DR_SHARD_SEND)
      r = ncclSend(at(buffer(local, op.buffer), op.src_offset), (size_t)op.bytes, ncclUint8, op.peer, comm->comm, st);
    else if (op.kind == DR_SHARD_RECV)
      r = ncclRecv(at(buffer(global, op.buffer), op.dst_offset), (size_t)op.bytes, ncclUint8, op.peer, comm->comm,
                   st);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_fail(r, op.kind == DR_SHARD_SEND ? "ncclSend" : "ncclRecv");
    }
  }
  r = ncclGroupEnd();
  return r == ncclSuccess ? DR_OK : nccl_fail(r, "ncclGroupEnd");
}

}  // extern "C"
