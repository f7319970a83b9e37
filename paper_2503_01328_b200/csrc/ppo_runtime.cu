// libppo_b200.so -- housekeeping, pinned host pool (K2), transfer slots (K2), pack (K1).
//
// The reference models these as quantities only: the payload bytes
// (pkg/src/ppoff/costs.py:99-105), the single-stream transfer slots
// (offload.py:133-220), host bins (offload.py:305-340) and residency
// (sim.py:462-487).  Here they are real copies on a dedicated copy stream.
#include <cuda.h>  // driver-API types only: entry points come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "ppo_common.cuh"

namespace ppo {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_error = buf;
  return code;
}

int cuda_error(cudaError_t err, const char* what) {
  return set_error((int)err, "%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
}

int pdl_mode() {
  static const int mode = [] {
    const char* e = std::getenv("PPO_PDL");
    return e ? std::atoi(e) : 0;
  }();
  return mode;
}

int sm_count_current() {
  static thread_local int cached_dev = -1, cached_sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      cached_sms = sms;
    cached_dev = dev;
  }
  return cached_sms;
}

// -------------------------------------------------------------------- K1 pack
constexpr int kMaxGather = 32;
struct GatherArgs {
  ppo_gather_item item[kMaxGather];
  int n;
};

// Persistent gather: every thread walks each item's 16-byte chunks with a grid
// stride, four independent 16 B loads in flight before the stores.
__global__ void __launch_bounds__(256) pack_kernel(GatherArgs args, uint8_t* __restrict__ dst) {
  pdl_wait();
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < args.n; ++i) {
    const ppo_gather_item it = args.item[i];
    const uint64_t row_chunks = it.row_bytes >> 4;
    const uint64_t total = row_chunks * it.rows;
    const uint64_t pitch = it.src_pitch ? it.src_pitch : it.row_bytes;
    const uint64_t dpitch = it.dst_pitch ? it.dst_pitch : it.row_bytes;
    const uint8_t* src = static_cast<const uint8_t*>(it.src);
    uint8_t* out = dst + it.dst_off;
    uint64_t c = tid;
    for (; c + 3 * nthr < total; c += 4 * nthr) {
      uint4 v[4];
      uint64_t dofs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint64_t cc = c + u * nthr;
        uint64_t r = cc / row_chunks, k = cc - r * row_chunks;
        v[u] = ld_stream(src + r * pitch + (k << 4));
        dofs[u] = r * dpitch + (k << 4);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) st_stream(out + dofs[u], v[u]);
    }
    for (; c < total; c += nthr) {
      uint64_t r = c / row_chunks, k = c - r * row_chunks;
      st_stream(out + r * dpitch + (k << 4), ld_stream(src + r * pitch + (k << 4)));
    }
  }
}

// TMA-staged pack for contiguous items: global -> shared (cp.async.bulk, mbarrier
// completion) -> global (cp.async.bulk store), kBulkStages chunks of kBulkChunk bytes
// in flight per CTA.  One thread per CTA issues everything; the copy engine-like TMA
// unit moves the bytes, so the SM's load/store pipes and registers stay idle.
constexpr int kBulkChunk = 16384;
constexpr int kBulkStages = 6;
struct BulkArgs {
  const uint8_t* src[kMaxGather];
  uint64_t dst_off[kMaxGather];
  uint64_t bytes[kMaxGather];
  uint64_t first_chunk[kMaxGather + 1];
  int n;
};

__global__ void __launch_bounds__(32) pack_bulk_kernel(BulkArgs a, uint8_t* __restrict__ dst) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bar[kBulkStages];
  if (threadIdx.x != 0) return;
  const uint64_t n_chunks = a.first_chunk[a.n];
  if (blockIdx.x >= n_chunks) return;
  const uint64_t mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  for (int i = 0; i < kBulkStages; ++i) mbar_init(&bar[i], 1);
  mbar_fence_init();
  auto locate = [&](uint64_t k, const uint8_t*& from, uint8_t*& to, uint32_t& len) {
    const uint64_t c = blockIdx.x + k * gridDim.x;
    int i = 0;
    while (c >= a.first_chunk[i + 1]) ++i;
    const uint64_t off = (c - a.first_chunk[i]) * kBulkChunk;
    const uint64_t rest = a.bytes[i] - off;
    from = a.src[i] + off;
    to = dst + a.dst_off[i] + off;
    len = (uint32_t)(rest < (uint64_t)kBulkChunk ? rest : (uint64_t)kBulkChunk);
  };
  auto load = [&](uint64_t k) {
    const uint8_t* from;
    uint8_t* to;
    uint32_t len;
    locate(k, from, to, len);
    const int sidx = (int)(k % kBulkStages);
    mbar_expect_tx(&bar[sidx], len);
    tma_load_1d(stage + sidx * kBulkChunk, from, len, &bar[sidx]);
  };
  for (uint64_t k = 0; k < mine && k < (uint64_t)kBulkStages; ++k) load(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const int sidx = (int)(k % kBulkStages);
    mbar_wait(&bar[sidx], (uint32_t)((k / kBulkStages) & 1));
    const uint8_t* from;
    uint8_t* to;
    uint32_t len;
    locate(k, from, to, len);
    tma_store_1d(to, stage + sidx * kBulkChunk, len);
    tma_store_commit();
    // refill the buffer the previous store read from, once that store is done reading
    if (k >= 1 && k - 1 + kBulkStages < mine) {
      tma_store_wait_read<1>();
      load(k - 1 + kBulkStages);
    }
  }
  tma_store_wait_all();
}

static bool pack_use_bulk() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("PPO_PACK_MODE");
    mode = (e && std::strcmp(e, "vector") == 0) ? 0 : 1;
  }
  return mode == 1;
}

}  // namespace ppo

using namespace ppo;

namespace {
__global__ void timestamp_kernel(unsigned long long* out) {
  pdl_wait();
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace

extern "C" {

int ppo_abi_version(void) { return PPO_ABI_VERSION; }

const char* ppo_last_error(void) { return t_error.c_str(); }

uint64_t ppo_kernel_launches(void) { return g_launches.load(); }

int ppo_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  if (!sm_count || !cc_major || !cc_minor) return set_error(PPO_EINVAL, "ppo_device_info: null output");
  PPO_TRY_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  PPO_TRY_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  PPO_TRY_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return PPO_OK;
}

// ------------------------------------------------------------------- pool
struct ppo_pool {
  void* base;
  uint64_t bytes;
  int numa_node;   // node the pages are bound to, -1: first touch (cudaHostAlloc)
  bool registered; // mmap + mbind + cudaHostRegister (else cudaHostAlloc)
};

// NUMA node of a GPU's PCI function (sysfs), -1 if unknown / not a NUMA system.
static int gpu_numa_node(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = (char)std::tolower(*c);
  char path[128];
  std::snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/numa_node", bus);
  FILE* f = std::fopen(path, "r");
  if (!f) return -1;
  int node = -1;
  if (std::fscanf(f, "%d", &node) != 1) node = -1;
  std::fclose(f);
  return node;
}

static int numa_nodes_online() {
  FILE* f = std::fopen("/sys/devices/system/node/online", "r");
  if (!f) return 1;
  int lo = 0, hi = 0;
  int n = std::fscanf(f, "%d-%d", &lo, &hi);
  std::fclose(f);
  return n == 2 ? hi - lo + 1 : 1;
}

static int pool_from_host_alloc(uint64_t bytes, ppo_pool* p) {
  void* base = nullptr;
  // Portable so every context of the process may DMA from it; pages land on the node
  // of the first-touching thread.
  PPO_TRY_CUDA(cudaHostAlloc(&base, bytes, cudaHostAllocPortable));
  p->base = base;
  p->bytes = bytes;
  p->numa_node = -1;
  p->registered = false;
  return PPO_OK;
}

int ppo_pool_create_numa(uint64_t bytes, int device, int numa_node, ppo_pool** out, int* node_out) {
  if (!out || bytes == 0) return set_error(PPO_EINVAL, "ppo_pool_create_numa: bad arguments");
  *out = nullptr;
  if (node_out) *node_out = -1;
  ppo_pool* p = static_cast<ppo_pool*>(std::calloc(1, sizeof(ppo_pool)));
  if (!p) return set_error(PPO_ENOMEM, "ppo_pool_create_numa: host malloc failed");
  int node = numa_node == -1 ? gpu_numa_node(device) : numa_node;
  if (node < 0 || numa_node == -2 || numa_nodes_online() < 2 || node >= 1024) {
    int rc = pool_from_host_alloc(bytes, p);
    if (rc != PPO_OK) {
      std::free(p);
      return rc;
    }
    *out = p;
    return PPO_OK;
  }
  // Bind the pages to the GPU's node BEFORE they are touched, touch them, then pin
  // them for the copy engines.  (A remote node halves the host-link rate a DMA
  // engine sees on 2-socket HGX boxes.)
  const long page = sysconf(_SC_PAGESIZE);
  const uint64_t len = (bytes + page - 1) / page * page;
  void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) {
    std::free(p);
    return set_error(PPO_ENOMEM, "ppo_pool_create_numa: mmap of %llu bytes failed", (unsigned long long)len);
  }
  unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
  mask[node / (8 * sizeof(unsigned long))] |= 1UL << (node % (8 * sizeof(unsigned long)));
  const int kMpolBind = 2;
  if (syscall(SYS_mbind, base, len, kMpolBind, mask, (unsigned long)1024, 0u) != 0) {
    munmap(base, len);
    std::free(p);
    return set_error(PPO_EINVAL, "ppo_pool_create_numa: mbind to node %d failed", node);
  }
  for (uint64_t off = 0; off < len; off += page) static_cast<volatile char*>(base)[off] = 0;  // fault in on `node`
  cudaError_t e = cudaHostRegister(base, len, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(base, len);
    std::free(p);
    return cuda_error(e, "cudaHostRegister");
  }
  p->base = base;
  p->bytes = len;
  p->numa_node = node;
  p->registered = true;
  if (node_out) *node_out = node;
  *out = p;
  return PPO_OK;
}

int ppo_pool_create(uint64_t bytes, ppo_pool** out) { return ppo_pool_create_numa(bytes, 0, -2, out, nullptr); }

int ppo_pool_destroy(ppo_pool* pool) {
  if (!pool) return PPO_OK;
  cudaError_t e = cudaSuccess;
  const bool registered = pool->registered;
  if (registered) {
    e = cudaHostUnregister(pool->base);
    munmap(pool->base, pool->bytes);
  } else {
    e = cudaFreeHost(pool->base);
  }
  std::free(pool);
  if (e != cudaSuccess) return cuda_error(e, registered ? "cudaHostUnregister" : "cudaFreeHost");
  return PPO_OK;
}

int ppo_pool_numa_node(const ppo_pool* pool) { return pool ? pool->numa_node : -1; }

void* ppo_pool_base(const ppo_pool* pool) { return pool ? pool->base : nullptr; }

uint64_t ppo_pool_bytes(const ppo_pool* pool) { return pool ? pool->bytes : 0; }

// --------------------------------------------------------------- K2 transfer
int ppo_transfer(int direction, const ppo_segment* segs, int nsegs, void* copy_stream, void* wait_event,
                 void* done_event) {
  if (direction != PPO_D2H && direction != PPO_H2D) return set_error(PPO_EINVAL, "ppo_transfer: bad direction");
  if (nsegs < 0 || (nsegs > 0 && !segs)) return set_error(PPO_EINVAL, "ppo_transfer: bad segments");
  cudaStream_t s = as_stream(copy_stream);
  if (wait_event) PPO_TRY_CUDA(cudaStreamWaitEvent(s, as_event(wait_event), 0));
  const cudaMemcpyKind kind = direction == PPO_D2H ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
  for (int i = 0; i < nsegs; ++i) {
    if (segs[i].bytes == 0) continue;
    if (!segs[i].dev || !segs[i].host) return set_error(PPO_EINVAL, "ppo_transfer: null segment %d", i);
    void* dst = direction == PPO_D2H ? segs[i].host : segs[i].dev;
    const void* src = direction == PPO_D2H ? segs[i].dev : segs[i].host;
    PPO_TRY_CUDA(cudaMemcpyAsync(dst, src, segs[i].bytes, kind, s));
  }
  if (done_event) PPO_TRY_CUDA(cudaEventRecord(as_event(done_event), s));
  return PPO_OK;
}

// ------------------------------------------- cross-rank transfer ordering (sync edges)
// Topology-synchronised plans (reference offload.py:223-248; honoured by sim.py:186-189)
// order transfers of two devices that share a PCIe switch.  On the GPU an edge is a
// 32-bit flag: the producer's copy stream writes 1 after its transfer, the consumer's
// copy stream waits for 1 (cuStreamWaitValue32, no host involvement, no SM) and resets
// it to 0.  Flags live in device memory (ranks in one process) or in host memory shared
// by the rank processes and mapped into each GPU's address space.
using WriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static int driver_fn(const char* name, void** fn) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn)
    return set_error(PPO_ENOTSUP, "driver entry point %s unavailable", name);
  return PPO_OK;
}

int ppo_stream_write_u32(void* stream, void* addr, uint32_t value) {
  static WriteValue32 fn = nullptr;
  if (!addr) return set_error(PPO_EINVAL, "ppo_stream_write_u32: null address");
  if (!fn) {
    void* p = nullptr;
    if (int rc = driver_fn("cuStreamWriteValue32", &p)) return rc;
    fn = reinterpret_cast<WriteValue32>(p);
  }
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value, 0);
  if (r != CUDA_SUCCESS) return set_error(PPO_ENOTSUP + 0, "cuStreamWriteValue32 failed (%d)", (int)r);
  return PPO_OK;
}

int ppo_stream_wait_u32(void* stream, void* addr, uint32_t value) {
  static WaitValue32 fn = nullptr;
  if (!addr) return set_error(PPO_EINVAL, "ppo_stream_wait_u32: null address");
  if (!fn) {
    void* p = nullptr;
    if (int rc = driver_fn("cuStreamWaitValue32", &p)) return rc;
    fn = reinterpret_cast<WaitValue32>(p);
  }
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                  CU_STREAM_WAIT_VALUE_EQ);
  if (r != CUDA_SUCCESS) return set_error(PPO_ENOTSUP, "cuStreamWaitValue32 failed (%d)", (int)r);
  return PPO_OK;
}

int ppo_host_register(void* ptr, uint64_t bytes, void** dev_ptr) {
  if (!ptr || !bytes || !dev_ptr) return set_error(PPO_EINVAL, "ppo_host_register: bad arguments");
  PPO_TRY_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  PPO_TRY_CUDA(cudaHostGetDevicePointer(dev_ptr, ptr, 0));
  return PPO_OK;
}

int ppo_host_unregister(void* ptr) {
  if (!ptr) return PPO_OK;
  PPO_TRY_CUDA(cudaHostUnregister(ptr));
  return PPO_OK;
}

int ppo_timestamp(uint64_t* slot, void* stream) {
  if (!slot) return set_error(PPO_EINVAL, "ppo_timestamp: null slot");
  launch_pdl(timestamp_kernel, 1, 1, 0, as_stream(stream), reinterpret_cast<unsigned long long*>(slot));
  PPO_LAUNCHED("timestamp_kernel");
  return PPO_OK;
}

// ------------------------------------------------------------------ K1 pack
int ppo_pack(const ppo_gather_item* items, int n, void* dst, void* stream) {
  if (n < 0 || n > kMaxGather || (n > 0 && (!items || !dst)))
    return set_error(PPO_EINVAL, "ppo_pack: bad arguments (n=%d, max %d)", n, kMaxGather);
  if (n == 0) return PPO_OK;
  if (!aligned16(dst)) return set_error(PPO_EINVAL, "ppo_pack: destination not 16-byte aligned");
  GatherArgs args;
  std::memset(&args, 0, sizeof(args));
  uint64_t chunks = 0;
  for (int i = 0; i < n; ++i) {
    const ppo_gather_item& it = items[i];
    const uint64_t pitch = it.src_pitch ? it.src_pitch : it.row_bytes;
    if (!it.src || !aligned16(it.src) || (it.dst_off & 15) || (it.row_bytes & 15) || (pitch & 15) ||
        (it.dst_pitch & 15))
      return set_error(PPO_EINVAL, "ppo_pack: item %d not 16-byte aligned", i);
    args.item[i] = it;
    chunks += (it.row_bytes >> 4) * it.rows;
  }
  args.n = n;
  if (chunks == 0) return PPO_OK;
  bool contiguous = true;
  for (int i = 0; i < n; ++i) {
    const ppo_gather_item& it = items[i];
    const uint64_t pitch = it.src_pitch ? it.src_pitch : it.row_bytes;
    const uint64_t dpitch = it.dst_pitch ? it.dst_pitch : it.row_bytes;
    contiguous &= it.rows <= 1 || (pitch == it.row_bytes && dpitch == it.row_bytes);
  }
  if (contiguous && pack_use_bulk() && (chunks << 4) >= (1u << 20)) {
    BulkArgs b;
    std::memset(&b, 0, sizeof(b));
    b.n = n;
    for (int i = 0; i < n; ++i) {
      b.src[i] = static_cast<const uint8_t*>(items[i].src);
      b.dst_off[i] = items[i].dst_off;
      b.bytes[i] = items[i].row_bytes * items[i].rows;
      b.first_chunk[i + 1] = b.first_chunk[i] + (b.bytes[i] + kBulkChunk - 1) / kBulkChunk;
    }
    static bool attr = false;
    const int smem = kBulkStages * kBulkChunk;
    if (!attr) {
      PPO_TRY_CUDA(cudaFuncSetAttribute(pack_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    const uint64_t cap = (uint64_t)sm_count_current() * 2;  // two 96 KB stagings per SM
    const uint64_t nc = b.first_chunk[n];
    const int blocks = (int)(nc < cap ? nc : cap);
    launch_pdl(pack_bulk_kernel, blocks, 32, smem, as_stream(stream), b, static_cast<uint8_t*>(dst));
    PPO_LAUNCHED("pack_bulk_kernel");
    return PPO_OK;
  }
  const int threads = 256;
  uint64_t want = (chunks + threads * 4 - 1) / (threads * 4);
  const uint64_t cap = (uint64_t)sm_count_current() * 8;  // 8 CTAs of 256 per SM resident
  const int blocks = (int)(want < cap ? (want ? want : 1) : cap);
  launch_pdl(pack_kernel, blocks, threads, 0, as_stream(stream), args, static_cast<uint8_t*>(dst));
  PPO_LAUNCHED("pack_kernel");
  return PPO_OK;
}

}  // extern "C"
