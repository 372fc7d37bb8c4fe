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
  std::vector<double*> xrecv;               // per rank: its kernel-exchange receive slots
  std::vector<unsigned long long*> xflag;   // per rank: its kernel-exchange flags
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

namespace {

__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned long long* p, unsigned long long v) {
  const unsigned long long t0 = global_ns();
  unsigned spins = 0;
  while (ld_acq_sys(p) < v) {
    if ((++spins & 1023u) == 0u && global_ns() - t0 > 20000000000ull) __trap();
    __nanosleep(64);
  }
}

struct PutArgs {
  long long plane, Nx, Ny, NzG, Klo, Khi;  // global plane indices of my bottom / top plane
  double* ylo;                             // my bottom plane (in y)
  double* yhi;                             // my top plane
  const double* xlo;                       // Dirichlet values (bcmode 1), may be null
  const double* xhi;
  double* put_lo;          // lower neighbour's receive slot for MY bottom plane (its "hi"), or null
  double* put_hi;          // upper neighbour's receive slot for MY top plane (its "lo"), or null
  unsigned long long* flag_lo;   // lower neighbour's "hi filled" flag
  unsigned long long* flag_hi;   // upper neighbour's "lo filled" flag
  const unsigned long long* cons_lo;  // lower / upper neighbour's "consumed" counter
  const unsigned long long* cons_hi;
  const double* recv_lo;   // my receive slots (this parity)
  const double* recv_hi;
  unsigned long long* my;  // my flags [lo filled, hi filled, consumed, -, up, down, barrier x2]
  unsigned long long seq;  // this exchange's number (1, 2, ...)
  int bcmode;
};

// Kernel-initiated interface exchange (§2.3 "NVSHMEM ... GPU-
// initiated communication"): (1) once the neighbour has
// consumed the previous use of this parity's slot, write my boundary planes
// straight into its receive slots through peer pointers (NVLink stores);
// (2) after a grid barrier (every block wrote and read my planes) block 0
// raises the neighbours' "filled" flags with a system-scope release; (3) every
// block waits for my own slots to be filled, then adds the received planes
// (Dirichlet rows re-imposed); (4) after a second barrier block 0 publishes
// "consumed".  Flags: [0] lo filled, [1] hi filled, [2] consumed, [4..5] the
// persistent CG's chain allreduce, [6..7] this kernel's grid barrier.
// Small cooperative grid: co-resident, and it leaves room for the other ranks'
// kernels when several ranks share one device (loopback).
__global__ void __launch_bounds__(256) plane_put_kernel(PutArgs P) {
  const long long st = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // the kernel's own self-resetting grid barrier in flags [6..7] (independent of
  // the exchange numbering, which the persistent CG kernel shares)
  GridBar* bar = reinterpret_cast<GridBar*>(P.my + 6);
  if (threadIdx.x == 0) {
    if (P.put_lo && P.seq > 2) spin_until(P.cons_lo, P.seq - 2);
    if (P.put_hi && P.seq > 2) spin_until(P.cons_hi, P.seq - 2);
  }
  __syncthreads();
  for (long long i = t0; i < P.plane; i += st) {
    if (P.put_lo) P.put_lo[i] = P.ylo[i];
    if (P.put_hi) P.put_hi[i] = P.yhi[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  grid_barrier(bar);  // every block's planes are written (and read)
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();
      if (P.put_lo) st_rel_sys(P.flag_lo, P.seq);
      if (P.put_hi) st_rel_sys(P.flag_hi, P.seq);
    }
    // neighbours' planes arrived
    if (P.put_lo) spin_until(P.my + 0, P.seq);
    if (P.put_hi) spin_until(P.my + 1, P.seq);
  }
  __syncthreads();
  for (long long i = t0; i < P.plane; i += st) {
    const long long I = i % P.Nx, J = i / P.Nx;
    const bool side = I == 0 || I == P.Nx - 1 || J == 0 || J == P.Ny - 1;
    if (P.put_lo) {
      double v = P.ylo[i] + P.recv_lo[i];
      if (P.bcmode && (side || P.Klo == 0 || P.Klo == P.NzG - 1))
        v = P.bcmode == 1 ? P.xlo[i] : (P.bcmode == 3 ? 1.0 : 0.0);
      P.ylo[i] = v;
    }
    if (P.put_hi) {
      double v = P.yhi[i] + P.recv_hi[i];
      if (P.bcmode && (side || P.Khi == 0 || P.Khi == P.NzG - 1))
        v = P.bcmode == 1 ? P.xhi[i] : (P.bcmode == 3 ? 1.0 : 0.0);
      P.yhi[i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  grid_barrier(bar);  // every block added its received planes
  if (blockIdx.x == 0 && threadIdx.x == 0) st_rel_sys(P.my + 2, P.seq);  // consumed
}

}  // namespace

// Kernel-initiated exchange: pointers of the neighbours' slots / flags.
hofem_status mesh_set_exchange(Mesh* m, int mode, cudaStream_t s) {
  if (mode != 0 && mode != 1) { set_error("hofem_mesh_set_exchange: mode 0 or 1"); return HOFEM_ERR_ARG; }
  if (m->nranks <= 1 || mode == m->xmode) { m->xmode = m->nranks > 1 ? mode : 0; return HOFEM_OK; }
  if (mode == 0) { m->xmode = 0; return HOFEM_OK; }
  const int r = m->rank, R = m->nranks;
  if (!m->d_xrecv) {
    // 2 parities x [lo | hi] planes, then the chain-allreduce slots (up, down)
    if (cudaMalloc(&m->d_xrecv, sizeof(double) * (4 * m->plane + 8)) != cudaSuccess ||
        cudaMalloc(&m->d_xflag, sizeof(unsigned long long) * 8) != cudaSuccess) {
      cudaGetLastError();
      set_error("hofem_mesh_set_exchange: out of device memory");
      return HOFEM_ERR_OOM;
    }
    HOFEM_CUDA(cudaMemsetAsync(m->d_xflag, 0, sizeof(unsigned long long) * 8, s));
    HOFEM_CUDA(cudaStreamSynchronize(s));
  }
  if (LoopGroup* g = m->comm->loop) {
    g->xrecv[r] = m->d_xrecv;
    g->xflag[r] = m->d_xflag;
    loop_barrier(g);
    for (int d = 0; d < 2; ++d) {
      const int q = d == 0 ? r - 1 : r + 1;
      m->peer_recv[d] = (q >= 0 && q < R) ? g->xrecv[q] : nullptr;
      m->peer_flag[d] = (q >= 0 && q < R) ? g->xflag[q] : nullptr;
      m->peer_ipc[d] = false;
    }
    loop_barrier(g);
  } else {
    // CUDA IPC handles of the receive slots and flags, swapped with the z
    // neighbours over NCCL, opened as peer pointers (NVLink between the GPUs)
    cudaIpcMemHandle_t h[2];
    HOFEM_CUDA(cudaIpcGetMemHandle(&h[0], m->d_xrecv));
    HOFEM_CUDA(cudaIpcGetMemHandle(&h[1], m->d_xflag));
    char* dsend = nullptr;
    char* drecv = nullptr;
    const size_t hb = sizeof(h);
    HOFEM_CUDA(cudaMalloc(&dsend, hb));
    HOFEM_CUDA(cudaMalloc(&drecv, 2 * hb));
    HOFEM_CUDA(cudaMemcpyAsync(dsend, h, hb, cudaMemcpyHostToDevice, s));
    ncclComm_t c = m->comm->nccl;
    HOFEM_TRY(nccl_status(ncclGroupStart(), "ncclGroupStart"));
    if (r > 0) {
      HOFEM_TRY(nccl_status(ncclSend(dsend, hb, ncclChar, r - 1, c, s), "ncclSend ipc"));
      HOFEM_TRY(nccl_status(ncclRecv(drecv, hb, ncclChar, r - 1, c, s), "ncclRecv ipc"));
    }
    if (r < R - 1) {
      HOFEM_TRY(nccl_status(ncclSend(dsend, hb, ncclChar, r + 1, c, s), "ncclSend ipc"));
      HOFEM_TRY(nccl_status(ncclRecv(drecv + hb, hb, ncclChar, r + 1, c, s), "ncclRecv ipc"));
    }
    HOFEM_TRY(nccl_status(ncclGroupEnd(), "ncclGroupEnd"));
    cudaIpcMemHandle_t nh[2][2];
    HOFEM_CUDA(cudaMemcpyAsync(nh, drecv, 2 * hb, cudaMemcpyDeviceToHost, s));
    HOFEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(dsend);
    cudaFree(drecv);
    for (int d = 0; d < 2; ++d) {
      const int q = d == 0 ? r - 1 : r + 1;
      if (q < 0 || q >= R) continue;
      void* pr = nullptr;
      void* pf = nullptr;
      HOFEM_CUDA(cudaIpcOpenMemHandle(&pr, nh[d][0], cudaIpcMemLazyEnablePeerAccess));
      HOFEM_CUDA(cudaIpcOpenMemHandle(&pf, nh[d][1], cudaIpcMemLazyEnablePeerAccess));
      m->peer_recv[d] = static_cast<double*>(pr);
      m->peer_flag[d] = static_cast<unsigned long long*>(pf);
      m->peer_ipc[d] = true;
    }
  }
  m->xmode = 1;
  return HOFEM_OK;
}

void mesh_release_exchange(Mesh* m) {
  for (int d = 0; d < 2; ++d) {
    if (m->peer_ipc[d]) {
      cudaIpcCloseMemHandle(m->peer_recv[d]);
      cudaIpcCloseMemHandle(m->peer_flag[d]);
    }
    m->peer_recv[d] = nullptr;
    m->peer_flag[d] = nullptr;
    m->peer_ipc[d] = false;
  }
  cudaFree(m->d_xrecv);
  cudaFree(m->d_xflag);
  m->d_xrecv = nullptr;
  m->d_xflag = nullptr;
}

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
  if (m->xmode == 1) {
    const unsigned long long seq = ++m->xseq;
    const long long par = (long long)(seq & 1ull) * 2 * plane;  // this parity's slots
    PutArgs P;
    P.plane = plane; P.Nx = m->Nx; P.Ny = m->Ny; P.NzG = m->NzG;
    P.Klo = (long long)m->p * m->z0;
    P.Khi = P.Klo + m->Nzl - 1;
    P.ylo = y; P.yhi = top;
    P.xlo = x; P.xhi = x ? x + (m->Nzl - 1) * plane : nullptr;
    P.put_lo = r > 0 ? m->peer_recv[0] + par + plane : nullptr;   // lower's "hi" slot
    P.put_hi = r < R - 1 ? m->peer_recv[1] + par : nullptr;       // upper's "lo" slot
    P.flag_lo = r > 0 ? m->peer_flag[0] + 1 : nullptr;
    P.flag_hi = r < R - 1 ? m->peer_flag[1] + 0 : nullptr;
    P.cons_lo = r > 0 ? m->peer_flag[0] + 2 : nullptr;
    P.cons_hi = r < R - 1 ? m->peer_flag[1] + 2 : nullptr;
    P.recv_lo = m->d_xrecv + par;
    P.recv_hi = m->d_xrecv + par + plane;
    P.my = m->d_xflag;
    P.seq = seq;
    P.bcmode = bcmode;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HOFEM_CUDA(cudaLaunchKernelEx(&cfg, plane_put_kernel, P));
    count_launch();
    return HOFEM_OK;
  }
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

hofem_status hofem_mesh_set_exchange(void* mesh, int mode, void* stream) {
  auto* m = static_cast<hofem::Mesh*>(mesh);
  if (!m) { hofem::set_error("hofem_mesh_set_exchange: NULL"); return HOFEM_ERR_ARG; }
  return hofem::mesh_set_exchange(m, mode, static_cast<cudaStream_t>(stream));
}

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
  g->xrecv.resize(nranks);
  g->xflag.resize(nranks);
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
