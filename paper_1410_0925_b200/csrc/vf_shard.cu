// Spatial sharding across GPUs (BASELINE config 5).
//
// Ownership: block b belongs to shard hash(b >> s) mod G, hashed on
// super-blocks of 2^s blocks per axis so shard seams rarely cut trilinear
// stencils.  Every shard marks all pixels but allocates only owned blocks
// (k_mark), integrates and raycasts its own blocks, and one exchange per
// frame composites the maps by nearest depth:
//   key(pixel) = float_bits(camera z of the hit) << 32 | rank   (UINT64_MAX: no hit)
//   keys  <- all_reduce(MIN)                      (positive float bits order like floats)
//   maps  <- all_reduce(SUM) of maps masked to the winning rank (x + 0 = x: exact)
// After the exchange every shard holds bit-identical maps, so the ICP of the
// next frame runs replicated and yields the identical pose on every shard
// without any per-iteration collective.
//
// Transports: NCCL (one process per GPU; the collectives are captured in the
// frame graph), or, for several shards living on one device (tests),
// k_shard_group_composite over the shards' buffers.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>

#include "vf_device.cuh"
#include "vf_kernels.h"

namespace vf {

__global__ void k_shard_keys(const float4* __restrict__ points, const FrameParams* __restrict__ fp, int npix, int rank,
                             unsigned long long* __restrict__ keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const float4 p = points[i];
  unsigned long long k = ~0ull;
  if (p.w != 0.0f) {
    const PoseD& w = fp->w2c;
    const double z = w.r[6] * p.x + w.r[7] * p.y + w.r[8] * p.z + w.t[2];
    const float zf = z > 0.0 ? (float)z : 0.0f;
    k = ((unsigned long long)__float_as_uint(zf) << 32) | (unsigned)rank;
  }
  keys[i] = k;
}

// Zero this shard's maps wherever another shard won (or nobody hit).
__global__ void k_shard_select(const unsigned long long* __restrict__ keys_min, int npix, int rank,
                               float4* __restrict__ points, float4* __restrict__ normals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const unsigned long long k = keys_min[i];
  if (k == ~0ull || (unsigned)(k & 0xffffffffu) != (unsigned)rank) {
    points[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    normals[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// In-process composite of n shards on one device: every shard receives the
// nearest hit (ties -> lowest rank).
__global__ void k_shard_group_composite(ShardGroupArgs g, int npix) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  unsigned long long best = ~0ull;
  for (int s = 0; s < g.n; ++s) {
    const unsigned long long k = g.keys[s][i];
    best = k < best ? k : best;
  }
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f), q = p;
  if (best != ~0ull) {
    const int w = (int)(best & 0xffffffffu);
    p = g.points[w][i];
    q = g.normals[w][i];
  }
  for (int s = 0; s < g.n; ++s) {
    g.points[s][i] = p;
    g.normals[s][i] = q;
  }
}

// ---------------------------------------------------------------------------
// Peer-memory composite (no NCCL): every shard publishes its per-pixel keys
// and reads the other shards' keys and winning map entries directly from
// their memory.  Per frame, on each shard's stream:
//   k_p2p_wait_done     -- before the raycast overwrites keys / maps: every
//                          shard finished reading the previous frame's;
//   raycast, k_shard_keys
//   k_p2p_signal_ready  -- frame number f into every shard's ready[rank]
//                          (release, system scope, after a system fence);
//   k_p2p_wait_ready    -- one thread waits for ready[r] >= f for all r (acquire);
//   k_p2p_composite     -- per pixel: min key over the shards, the winner's point
//                          and normal into this shard's maps (its own pixels
//                          untouched, so readers never race with writers);
//   k_p2p_signal_done   -- f into every shard's done[rank].
// Every shard ends with the identical maps the NCCL path produces.  A shard
// that does not answer within ~0.5 s counts as "no hit" and raises
// kErrShardXchg instead of hanging the frame.
namespace {
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// wait until flags[base + r] >= seq for every shard r; returns the mask of shards that answered
__device__ unsigned wait_all(const P2PArgs& a, int base, unsigned long long seq) {
  const unsigned long long* own = a.flags[a.rank];
  unsigned ok = 0;
  for (int r = 0; r < a.n; ++r) {
    for (long spin = 0;; ++spin) {
      if (ld_acquire_sys(own + base + r) >= seq) {
        ok |= 1u << r;
        break;
      }
      if (spin > (1l << 22)) {
        atomicOr(&a.ctr->error_flags, kErrShardXchg);
        break;
      }
      __nanosleep(64);
    }
  }
  return ok;
}
}  // namespace

__global__ void k_p2p_wait_done(P2PArgs a) {
  if (threadIdx.x != 0) return;
  const unsigned long long seq = a.flags[a.rank][kP2PSeq];  // the previous frame (0: none)
  if (seq > 0) wait_all(a, kP2PDone, seq);
}

__global__ void k_p2p_signal_ready(P2PArgs a) {
  if (threadIdx.x != 0) return;
  unsigned long long* own = a.flags[a.rank];
  const unsigned long long seq = own[kP2PSeq] + 1;
  own[kP2PSeq] = seq;
  __threadfence_system();  // this shard's keys and maps before the flag
  for (int r = 0; r < a.n; ++r) st_release_sys(a.flags[r] + kP2PReady + a.rank, seq);
}

// One thread waits (a full grid of spinning CTAs would starve the other
// shards' kernels when shards share a device); the answer mask goes to the
// composite through the flags area.
__global__ void k_p2p_wait_ready(P2PArgs a) {
  if (threadIdx.x != 0) return;
  unsigned long long* own = a.flags[a.rank];
  own[kP2PMask] = wait_all(a, kP2PReady, own[kP2PSeq]);
}

__global__ void k_p2p_composite(P2PArgs a, float4* __restrict__ points, float4* __restrict__ normals, int npix) {
  const unsigned ok = (unsigned)a.flags[a.rank][kP2PMask];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += gridDim.x * blockDim.x) {
    unsigned long long best = ~0ull;
    for (int r = 0; r < a.n; ++r) {
      if (!((ok >> r) & 1u)) continue;
      const unsigned long long k = __ldcv(a.keys[r] + i);
      best = k < best ? k : best;
    }
    const int w = best == ~0ull ? -1 : (int)(best & 0xffffffffu);
    if (w == a.rank) continue;  // this shard's own hit stays (and may be read by the others)
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f), q = p;
    if (w >= 0) {
      p = __ldcv(a.points[w] + i);
      q = __ldcv(a.normals[w] + i);
    }
    points[i] = p;
    normals[i] = q;
  }
}

__global__ void k_p2p_signal_done(P2PArgs a) {
  if (threadIdx.x != 0) return;
  const unsigned long long seq = a.flags[a.rank][kP2PSeq];
  __threadfence_system();
  for (int r = 0; r < a.n; ++r) st_release_sys(a.flags[r] + kP2PDone + a.rank, seq);
}

}  // namespace vf

// ---------------------------------------------------------------------------
// NCCL, loaded at run time: the process may already carry another libnccl
// (PyTorch's); reuse whichever is loaded, else the system library.
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // one already in the process (PyTorch's) first, then VF_NCCL_LIB, then the system's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && std::getenv("VF_NCCL_LIB")) h = dlopen(std::getenv("VF_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy;
    return a;
  }();
  return api;
}

}  // namespace

namespace vf {

int nccl_unique_id(void* out) {
  NcclApi& a = nccl();
  if (!a.ok) return -1;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return -2;
  memcpy(out, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(void** comm, const void* id_bytes, int nranks, int rank) {
  NcclApi& a = nccl();
  if (!a.ok) return -1;
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, nranks, id, rank);
  if (r != ncclSuccess) {
    std::fprintf(stderr, "[voxfuse_b200] ncclCommInitRank: %s\n", a.error_string ? a.error_string(r) : "?");
    return -2;
  }
  *comm = c;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

// keys -> all_reduce(MIN) -> select -> all_reduce(SUM) of both maps, on `st`.
int nccl_composite(void* comm, cudaStream_t st, const FrameParams* fp, float4* points, float4* normals,
                   unsigned long long* keys, int npix, int rank) {
  NcclApi& a = nccl();
  if (!a.ok || !comm) return -1;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const int blocks = (npix + 255) / 256;
  k_shard_keys<<<blocks, 256, 0, st>>>(points, fp, npix, rank, keys);
  if (a.all_reduce(keys, keys, (size_t)npix, ncclUint64, ncclMin, c, st) != ncclSuccess) return -2;
  k_shard_select<<<blocks, 256, 0, st>>>(keys, npix, rank, points, normals);
  if (a.all_reduce(points, points, (size_t)npix * 4, ncclFloat32, ncclSum, c, st) != ncclSuccess) return -2;
  if (a.all_reduce(normals, normals, (size_t)npix * 4, ncclFloat32, ncclSum, c, st) != ncclSuccess) return -2;
  return 0;
}

}  // namespace vf
