// comm.cu -- the parallel prolongation/restriction P, P^T of the paper's triple
// product P^T A P (§2.3), collapsed for a z-slab partition into
// one exchange per apply: each rank sends its two boundary
// lattice planes (contiguous in the x-fastest layout, so no pack kernel) to its
// z-neighbours with grouped ncclSend/ncclRecv over NVLink, then adds what it
// received.  a+b == b+a in IEEE arithmetic, so both copies of a shared plane end
// bitwise identical (reading R9).  Dirichlet rows on the planes are re-imposed
// after the sum.  CG dot products use ncclAllReduce of one FP64 (§8(e)).
#include <condition_variable>
#include <mutex>
#include <vector>

#include "internal.h"

namespace hofem {

struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<cudaEvent_t> ev_a, ev_b;      // per rank: "my data is ready" / "I am done reading"
  std::vector<const double*> lo, hi;        // per rank: its bottom / top plane this exchange
  double* slots = nullptr;                  // allreduce staging, n * kSlot doubles
  static constexpr int kSlot = 8;
  int attached = 0;
};

namespace {

void loop_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  const long long my = g->gen;
  if (++g->arrived == g->n) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->gen != my; });
  }
}

}  // namespace

namespace {

__global__ void add_plane_kernel(long long plane, long long Nx, long long Ny, long long Kg,
                                 long long NzG, int bcmode, const double* __restrict__ xbc,
                                 const double* __restrict__ recv, double* __restrict__ y) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= plane) return;
  double v = y[t] + recv[t];
  if (bcmode) {
    long long I = t % Nx, J = t / Nx;
    if (I == 0 || I == Nx - 1 || J == 0 || J == Ny - 1 || Kg == 0 || Kg == NzG - 1)
      v = bcmode == 1 ? xbc[t] : (bcmode == 3 ? 1.0 : 0.0);
  }
  y[t] = v;
}

hofem_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HOFEM_OK;
  set_error("%s: %s", what, ncclGetErrorString(r));
  return HOFEM_ERR_NCCL;
}

}  // namespace

hofem_status exchange_planes(Op* op, const double* x, double* y, cudaStream_t s) {
  return exchange_planes_bc(op, x, y, op->bc ? (x ? 1 : 2) : 0, s);
}

// bcmode on the summed planes' Dirichlet points: 0 none, 1 y = x, 2 y = 0, 3 y = 1
hofem_status exchange_planes_bc(Op* op, const double* x, double* y, int bcmode, cudaStream_t s) {
  Mesh* m = op->mesh;
  if (m->nranks <= 1) return HOFEM_OK;
  const long long plane = m->plane;
  const int r = m->rank, R = m->nranks;
  double* top = y + (m->Nzl - 1) * plane;
  if (LoopGroup* g = m->comm->loop) {
    // loopback: publish my planes, copy the neighbours' once they are ready,
    // and modify mine only after the neighbours have copied them
    g->lo[r] = y;
    g->hi[r] = top;
    HOFEM_CUDA(cudaEventRecord(g->ev_a[r], s));
    loop_barrier(g);
    if (r > 0) {
      HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_a[r - 1], 0));
      HOFEM_CUDA(cudaMemcpyAsync(m->d_recv, g->hi[r - 1], sizeof(double) * plane,
                                 cudaMemcpyDeviceToDevice, s));
    }
    if (r < R - 1) {
      HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_a[r + 1], 0));
      HOFEM_CUDA(cudaMemcpyAsync(m->d_recv + plane, g->lo[r + 1], sizeof(double) * plane,
                                 cudaMemcpyDeviceToDevice, s));
    }
    HOFEM_CUDA(cudaEventRecord(g->ev_b[r], s));
    loop_barrier(g);
    if (r > 0) HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_b[r - 1], 0));
    if (r < R - 1) HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_b[r + 1], 0));
  } else {
  ncclComm_t c = m->comm->nccl;
  HOFEM_TRY(nccl_status(ncclGroupStart(), "ncclGroupStart"));
  if (r > 0) {
    HOFEM_TRY(nccl_status(ncclSend(y, plane, ncclDouble, r - 1, c, s), "ncclSend lo"));
    HOFEM_TRY(nccl_status(ncclRecv(m->d_recv, plane, ncclDouble, r - 1, c, s), "ncclRecv lo"));
  }
  if (r < R - 1) {
    HOFEM_TRY(nccl_status(ncclSend(top, plane, ncclDouble, r + 1, c, s), "ncclSend hi"));
    HOFEM_TRY(nccl_status(ncclRecv(m->d_recv + plane, plane, ncclDouble, r + 1, c, s),
                          "ncclRecv hi"));
  }
  HOFEM_TRY(nccl_status(ncclGroupEnd(), "ncclGroupEnd"));
  }
  const unsigned g = (unsigned)((plane + 255) / 256);
  const long long K0 = (long long)m->p * m->z0;
  if (r > 0) {
    add_plane_kernel<<<g, 256, 0, s>>>(plane, m->Nx, m->Ny, K0, m->NzG, bcmode, x, m->d_recv, y);
    HOFEM_LAUNCHED();
  }
  if (r < R - 1) {
    add_plane_kernel<<<g, 256, 0, s>>>(plane, m->Nx, m->Ny, K0 + m->Nzl - 1, m->NzG, bcmode,
                                       x ? x + (m->Nzl - 1) * plane : nullptr,
                                       m->d_recv + plane, top);
    HOFEM_LAUNCHED();
  }
  return HOFEM_OK;
}

namespace {
// d_val[i] = sum over ranks (rank order) of the staged values
__global__ void loop_sum_kernel(const double* __restrict__ slots, int n, int count, int stride,
                                double* __restrict__ d_val) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < n; ++r) s += slots[r * stride + i];
  d_val[i] = s;
}
}  // namespace

hofem_status allreduce_sum(Mesh* m, double* d_val, int count, cudaStream_t s) {
  if (m->nranks <= 1) return HOFEM_OK;
  if (LoopGroup* g = m->comm->loop) {
    if (count > LoopGroup::kSlot) {
      set_error("loopback allreduce: count %d > %d", count, LoopGroup::kSlot);
      return HOFEM_ERR_ARG;
    }
    const int r = m->rank;
    HOFEM_CUDA(cudaMemcpyAsync(g->slots + r * LoopGroup::kSlot, d_val, sizeof(double) * count,
                               cudaMemcpyDeviceToDevice, s));
    HOFEM_CUDA(cudaEventRecord(g->ev_a[r], s));
    loop_barrier(g);
    for (int q = 0; q < g->n; ++q)
      if (q != r) HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_a[q], 0));
    loop_sum_kernel<<<1, 32, 0, s>>>(g->slots, g->n, count, LoopGroup::kSlot, d_val);
    HOFEM_LAUNCHED();
    HOFEM_CUDA(cudaEventRecord(g->ev_b[r], s));
    loop_barrier(g);
    for (int q = 0; q < g->n; ++q)
      if (q != r) HOFEM_CUDA(cudaStreamWaitEvent(s, g->ev_b[q], 0));
    return HOFEM_OK;
  }
  return nccl_status(
      ncclAllReduce(d_val, d_val, count, ncclDouble, ncclSum, m->comm->nccl, s), "ncclAllReduce");
}

}  // namespace hofem

extern "C" {

hofem_status hofem_comm_unique_id(void* out) {
  if (!out) { hofem::set_error("hofem_comm_unique_id: NULL"); return HOFEM_ERR_ARG; }
  ncclUniqueId id;
  HOFEM_TRY(hofem::nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId"));
  static_assert(sizeof(id) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(out, &id, sizeof(id));
  return HOFEM_OK;
}

hofem_status hofem_comm_init(const void* nccl_id, int rank, int nranks, int device,
                             void** comm_out) {
  if (!nccl_id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) {
    hofem::set_error("hofem_comm_init: bad arguments");
    return HOFEM_ERR_ARG;
  }
  HOFEM_CUDA(cudaSetDevice(device));
  auto* c = new hofem::Comm();
  c->rank = rank; c->nranks = nranks; c->device = device;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  hofem_status st = hofem::nccl_status(ncclCommInitRank(&c->nccl, nranks, id, rank),
                                       "ncclCommInitRank");
  if (st != HOFEM_OK) { delete c; return st; }
  *comm_out = c;
  return HOFEM_OK;
}

void hofem_comm_destroy(void* comm) {
  auto* c = static_cast<hofem::Comm*>(comm);
  if (!c) return;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

hofem_status hofem_loopback_group_create(int nranks, void** group_out) {
  if (nranks < 1 || !group_out) {
    hofem::set_error("hofem_loopback_group_create: bad arguments");
    return HOFEM_ERR_ARG;
  }
  auto* g = new hofem::LoopGroup();
  g->n = nranks;
  g->ev_a.resize(nranks);
  g->ev_b.resize(nranks);
  g->lo.resize(nranks);
  g->hi.resize(nranks);
  for (int r = 0; r < nranks; ++r) {
    if (cudaEventCreateWithFlags(&g->ev_a[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_b[r], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      hofem::set_error("hofem_loopback_group_create: event creation failed");
      return HOFEM_ERR_CUDA;
    }
  }
  if (cudaMalloc(&g->slots, sizeof(double) * nranks * hofem::LoopGroup::kSlot) != cudaSuccess) {
    cudaGetLastError();
    hofem::set_error("hofem_loopback_group_create: out of device memory");
    return HOFEM_ERR_OOM;
  }
  *group_out = g;
  return HOFEM_OK;
}

hofem_status hofem_comm_init_loopback(void* group, int rank, void** comm_out) {
  auto* g = static_cast<hofem::LoopGroup*>(group);
  if (!g || !comm_out || rank < 0 || rank >= g->n) {
    hofem::set_error("hofem_comm_init_loopback: bad arguments");
    return HOFEM_ERR_ARG;
  }
  auto* c = new hofem::Comm();
  c->rank = rank;
  c->nranks = g->n;
  cudaGetDevice(&c->device);
  c->loop = g;
  *comm_out = c;
  return HOFEM_OK;
}

void hofem_loopback_group_destroy(void* group) {
  auto* g = static_cast<hofem::LoopGroup*>(group);
  if (!g) return;
  for (auto e : g->ev_a) cudaEventDestroy(e);
  for (auto e : g->ev_b) cudaEventDestroy(e);
  cudaFree(g->slots);
  delete g;
}

}  // extern "C"
