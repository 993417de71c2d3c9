/*
 * dr_shard.h — mesh sharding across GPUs and the fragment gather.
 *
 * The reference processes the meshes of a batch one after another and nothing crosses meshes
 * (/root/reference/proj/src/mesh_raster.cpp:240-283 forward, :380-401 backward per face range), so a batch
 * shards by mesh: each rank calls dr_rasterize_meshes_fwd/_bwd (dr_raster.h) with the GLOBAL face ranges
 * (mesh_to_face_first_idx / num_faces_per_mesh) of its own meshes over the whole packed face_verts. Its
 * pix_to_face then holds global packed face ids and its backward writes only its meshes' rows of
 * grad_face_verts; the data path needs no collective. The only exchange is the optional gather of the per-mesh
 * outputs to one rank over NVLink:
 *
 *   libdr_raster_b200.so  dr_shard_plan_lpt, dr_shard_gather_ops   (host logic; no NCCL dependency)
 *   libdr_shard_b200.so   dr_shard_comm_*, dr_shard_gather          (executes the op list with NCCL: one
 *                                                                    ncclGroupStart/End of ncclSend/ncclRecv
 *                                                                    plus device copies for the root's meshes)
 *
 * Buffers of a gather (all device pointers):
 *   local  fragments of this rank's meshes [n_local, H, W, K(,3)] in local_index order; grad_face_verts the
 *          whole [F,3,3] array (this rank's rows written by its backward)
 *   global (root only) fragments [N, H, W, K(,3)] in global mesh order; grad_face_verts [F,3,3]
 * A call gathers the meshes whose local_index lies in [local_lo, local_hi) on every rank, so a caller that
 * computes its meshes in groups can gather each group while the next one computes (pipelining).
 */
#ifndef DR_SHARD_H
#define DR_SHARD_H

#include <stdint.h>

#include "dr_raster.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { DR_SHARD_SEND = 0, DR_SHARD_RECV = 1, DR_SHARD_COPY = 2 };
enum { DR_BUF_P2F = 0, DR_BUF_ZBUF = 1, DR_BUF_BARY = 2, DR_BUF_DISTS = 3, DR_BUF_GRAD = 4 };

/* One transfer of a gather: SEND local[buffer] + src_offset -> peer (the root); RECV from peer into
 * global[buffer] + dst_offset; COPY local -> global on the root (its own meshes; skipped when the two
 * addresses coincide, e.g. a shared grad_face_verts array). Offsets and sizes in bytes. */
typedef struct dr_shard_op {
  int32_t kind, peer, buffer, mesh;
  int64_t src_offset, dst_offset, bytes;
} dr_shard_op;

/* Longest-processing-time assignment of N meshes to nranks ranks by cost (face count): meshes by decreasing
 * cost (ties: lower index) each to the least-loaded rank (ties: lower rank). owner[m] = rank, local_index[m] =
 * position of m in its owner's ascending mesh list. Host arrays. */
int dr_shard_plan_lpt(const int64_t* costs, int64_t N, int32_t nranks, int32_t* owner, int32_t* local_index);

/* The transfers `rank` takes part in when the meshes with local_index in [local_lo, local_hi) are gathered to
 * `root`: sends of its meshes (rank != root), receives of the other ranks' meshes and copies of its own
 * (rank == root). Every rank derives the same sequence per (sender, root) pair from the same plan, which is
 * how sends and receives match. payload_bytes = 4 (fp32 zbuf/bary/dists) or 8 (fp64); with_grad adds the
 * meshes' grad_face_verts rows (mesh_first / mesh_num: host copies of the global face ranges).
 * Writes at most cap ops (ops may be NULL to count) and the number needed to *n_ops. */
int dr_shard_gather_ops(int64_t N, const int32_t* owner, const int32_t* local_index, const int64_t* mesh_first,
                        const int64_t* mesh_num, int64_t slots_per_mesh, int32_t payload_bytes, int32_t with_grad,
                        int32_t nranks, int32_t rank, int32_t root, int32_t local_lo, int32_t local_hi,
                        dr_shard_op* ops, int64_t cap, int64_t* n_ops);

/* ---- libdr_shard_b200.so: NCCL executor ---- */
typedef struct dr_shard_comm* dr_shard_comm_t;

typedef struct dr_shard_buffers {
  void* pix_to_face;
  void* zbuf;
  void* bary;
  void* dists;
  void* grad_face_verts; /* may be NULL when with_grad = 0 */
} dr_shard_buffers;

/* ncclGetUniqueId on one rank; the 128 bytes travel to the others out of band (torch.distributed). */
int dr_shard_unique_id(uint8_t id[128]);
/* ncclCommInitRank on the current CUDA device. */
int dr_shard_comm_init(int32_t nranks, int32_t rank, const uint8_t id[128], dr_shard_comm_t* comm);
int dr_shard_comm_destroy(dr_shard_comm_t comm);
/* Gather (see dr_shard_gather_ops) as ONE NCCL group of ncclSend / ncclRecv on `stream`, plus the root's
 * device copies of its own meshes. Stream-ordered: the caller orders it after the producing kernels (e.g. an
 * event) and may run it on a side stream so it overlaps the next group's compute. `global` is read on the
 * root only. */
int dr_shard_gather(dr_shard_comm_t comm, int32_t root, int64_t N, const int32_t* owner, const int32_t* local_index,
                    const int64_t* mesh_first, const int64_t* mesh_num, int64_t slots_per_mesh,
                    int32_t payload_bytes, int32_t with_grad, int32_t local_lo, int32_t local_hi,
                    const dr_shard_buffers* local, const dr_shard_buffers* global, dr_stream_t stream);
/* Message of the last failing dr_shard_* call of libdr_shard_b200.so on this thread. */
const char* dr_shard_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DR_SHARD_H */
