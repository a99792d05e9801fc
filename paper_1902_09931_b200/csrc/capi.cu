// capi.cu — the extern "C" boundary (include/stengrid/sg.h): stencil plans,
// grid helpers, error reporting. Validation order and messages follow the
// reference's create_plan / validate_kind / make_tiles / compute
// (stencil.cpp:128-235, grid.cpp:42-82) so the C++ layer can rethrow the
// same exception types for the same conditions.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "sg_internal.hpp"

namespace {

thread_local std::string t_msg;
thread_local int t_system = -1;

template <typename F>
sg_status guard(F&& f) {
  try {
    f();
    return SG_OK;
  } catch (const sg::Error& e) {
    t_msg = e.what();
    t_system = e.system;
    return e.status;
  } catch (const std::exception& e) {
    t_msg = e.what();
    return SG_ERR_CUDA;
  }
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw sg::Error(SG_ERR_NO_DEVICE, "stengrid: no CUDA device visible (there is no CPU fallback)");
}

std::vector<std::pair<int, int>> tiles_for(int ny, int numTiles) {
  // make_tiles, grid.cpp:62-82
  if (ny < 1) sg::invalid("make_tiles: ny must be >= 1");
  if (numTiles < 1 || numTiles > ny)
    sg::invalid("make_tiles: numTiles must satisfy 1 <= numTiles <= ny");
  std::vector<std::pair<int, int>> t;
  const int base = ny / numTiles, extra = ny % numTiles;
  int j = 0;
  for (int k = 0; k < numTiles; ++k) {
    const int rows = base + (k < extra ? 1 : 0);
    t.emplace_back(j, j + rows);
    j += rows;
  }
  return t;
}

// numWorkers -> GPU count. 0 ("clip", the default): G = min(numWorkers,
// visible GPUs) — a reference caller passing its host thread count gets every
// GPU and no oversubscription. 1 ("modulo"): G = numWorkers, worker w on
// device w % GPUs — several workers share a device (tests of the multi-GPU
// path on a one-GPU box). SG_DEVICE_MAP=modulo selects 1 at load.
std::atomic<int> g_device_map{-1};
int device_map() {
  int m = g_device_map.load();
  if (m < 0) {
    const char* e = std::getenv("SG_DEVICE_MAP");
    m = e && std::strcmp(e, "modulo") == 0 ? 1 : 0;
    g_device_map.store(m);
  }
  return m;
}

}  // namespace

struct sg_plan_s {
  bool valid = false;
  sg_direction dir = SG_DIR_X;
  sg_boundary mode = SG_PERIODIC;
  sg_extents ext{};
  int fn = SG_FN_NONE;
  std::vector<double> values;
  sg_dtype dtype = SG_F64;
  int nx = 0, ny = 0;
  sg_memory memory = SG_MEM_HOST;
  int numTiles = 1, numWorkers = 1;
  std::vector<std::pair<int, int>> tiles;
  int device = 0;
  cudaStream_t stream = nullptr;
  struct Buf {
    void* host = nullptr;
    void* dev = nullptr;
    bool owned = false;     // device mirror allocated by the plan
    bool devValid = false;  // device copy holds the current values
    bool hostValid = true;  // host copy holds the current values
    bool halosValid = false;  // multi-worker: the slabs' halo rows match their owners' rows
  } buf[2];
  int inIdx = 0;
  // Host-pipelining resources (Residency::Host on large periodic grids).
  cudaStream_t sH2D = nullptr, sD2H = nullptr;
  std::vector<cudaEvent_t> events;
  bool registered[2] = {false, false};
  // numWorkers -> GPUs (host grids only): worker w owns make_tiles(ny, G)'s
  // w-th row block on device `device`, both bindings stored as ext slabs
  // [top halo | own rows | bottom halo]. Empty: single-device plan.
  struct Worker {
    int device = 0;
    int r0 = 0, r1 = 0;
    cudaStream_t stream = nullptr, sH2D = nullptr, sD2H = nullptr;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;
    std::vector<cudaEvent_t> ev;  // pipeline events
    int own() const { return r1 - r0; }
  };
  std::vector<Worker> workers;
  // Streamed (out-of-core) host plan: no full-size device mirrors; every
  // compute() streams the grid through a ring of NSLOT row-chunk buffers
  // (chunkRows output rows + top/bottom halo rows each) — host grids larger
  // than the device's memory work, as the paper's tiling intended
  // (PAPER.md:120-129). Chosen when the two mirrors would not fit in free
  // device memory (SG_STREAM_PLANS=1 forces it; SG_STREAM_ROWS sets the
  // chunk height).
  static constexpr int NSLOT = 3;
  bool streamed = false;
  int chunkRows = 0;
  struct Slot {
    void* in = nullptr;
    void* out = nullptr;
    cudaEvent_t loaded = nullptr, computed = nullptr, drained = nullptr;
    bool used = false;
  } slots[NSLOT];

  size_t elem() const { return dtype == SG_F64 ? 8 : 4; }
  size_t bytes() const { return static_cast<size_t>(nx) * ny * (dtype == SG_F64 ? 8 : 4); }

  void release() {
    if (!valid) return;
    for (auto& w : workers) {
      cudaSetDevice(w.device);
      if (w.stream) cudaStreamSynchronize(w.stream);
      for (void* b : w.buf)
        if (b) cudaFree(b);
      for (auto e : w.ev) cudaEventDestroy(e);
      if (w.done) cudaEventDestroy(w.done);
      for (cudaStream_t t : {w.stream, w.sH2D, w.sD2H})
        if (t) cudaStreamDestroy(t);
    }
    workers.clear();
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (sD2H) cudaStreamSynchronize(sD2H);
    for (auto& sl : slots) {
      if (sl.in) cudaFree(sl.in);
      if (sl.out) cudaFree(sl.out);
      for (cudaEvent_t e : {sl.loaded, sl.computed, sl.drained})
        if (e) cudaEventDestroy(e);
      sl = Slot{};
    }
    streamed = false;
    for (auto& b : buf)
      if (b.owned && b.dev) cudaFree(b.dev);
    for (int k = 0; k < 2; ++k)
      if (registered[k]) cudaHostUnregister(buf[k].host);
    for (auto e : events) cudaEventDestroy(e);
    events.clear();
    if (sH2D) cudaStreamDestroy(sH2D);
    if (sD2H) cudaStreamDestroy(sD2H);
    sH2D = sD2H = nullptr;
    registered[0] = registered[1] = false;
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    buf[0] = Buf{};
    buf[1] = Buf{};
    tiles.clear();
    values.clear();
    valid = false;
  }
};

static void setup_workers(sg_plan_s* p, int G, int ndev);

// The slot ring of a streamed compute (streamed plans, and large
// non-periodic Residency::Host computes of mirrored plans): chunk height
// SG_STREAM_ROWS, else ~128 MiB of output rows, at least one row.
static void setup_streaming(sg_plan_s* p) {
  const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
  const int H = p->ext.top + p->ext.bottom;
  int rows = 0;
  if (const char* e = std::getenv("SG_STREAM_ROWS")) rows = std::atoi(e);
  if (rows <= 0) rows = static_cast<int>(std::max<size_t>(1, (128ull << 20) / rowB));
  rows = std::min(rows, p->ny);
  p->chunkRows = rows;
  for (auto& sl : p->slots) {
    SG_CUDA(cudaMalloc(&sl.in, (static_cast<size_t>(rows) + H) * rowB));
    SG_CUDA(cudaMalloc(&sl.out, static_cast<size_t>(rows) * rowB));
    for (cudaEvent_t* e : {&sl.loaded, &sl.computed, &sl.drained})
      SG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
}

extern "C" {

sg_status sg_internal_set_error(const char* msg, int system) {
  t_msg = msg;
  t_system = system;
  return SG_OK;
}

int sg_abi_version(void) { return SG_ABI_VERSION; }
const char* sg_last_error(void) { return t_msg.c_str(); }
int sg_last_error_system(void) { return t_system; }
uint64_t sg_launch_count(void) { return sg::g_launches.load(); }

sg_status sg_init(int device) {
  return guard([&] {
    require_device();
    SG_CUDA(cudaSetDevice(device));
    SG_CUDA(cudaFree(nullptr));
  });
}

int sg_function_min_coe(int fn) {
  int w, h, c;
  return sg::function_shape(fn, &w, &h, &c) ? c : -1;
}
const char* sg_function_name(int fn) { return sg::function_name(fn); }

sg_status sg_wrap(int64_t i, int n, int* out) {
  return guard([&] {
    if (n <= 0) sg::invalid("wrap: period must be >= 1");
    int64_t r = i % n;
    if (r < 0) r += n;
    *out = static_cast<int>(r);
  });
}

sg_status sg_make_tiles(int ny, int numTiles, int* begins, int* ends) {
  return guard([&] {
    const auto t = tiles_for(ny, numTiles);
    for (size_t k = 0; k < t.size(); ++k) {
      begins[k] = t[k].first;
      ends[k] = t[k].second;
    }
  });
}

sg_status sg_plan_create(sg_direction dir, sg_boundary mode, sg_extents ext, sg_function fn,
                         const double* values, size_t count, sg_dtype dtype, void* in, void* out,
                         int nx, int ny, sg_memory memory, int numTiles, int numWorkers,
                         sg_plan_t* plan) {
  return guard([&] {
    if (!plan) sg::invalid("create_plan: null plan handle");
    *plan = nullptr;
    if (nx < 1 || ny < 1) sg::invalid("Grid2D: nx and ny must be >= 1");
    if (dtype != SG_F64 && dtype != SG_F32) sg::invalid("create_plan: unknown dtype");
    if (dir != SG_DIR_X && dir != SG_DIR_Y && dir != SG_DIR_XY)
      sg::invalid("create_plan: unknown direction");
    if (mode != SG_PERIODIC && mode != SG_NONPERIODIC) sg::invalid("create_plan: unknown boundary mode");
    // stencil.cpp:156-157
    if (in == out || in == nullptr || out == nullptr)
      sg::invalid("create_plan: input and output must be distinct buffers");
    // validate_kind, stencil.cpp:128-148
    if (ext.left < 0 || ext.right < 0 || ext.top < 0 || ext.bottom < 0)
      sg::invalid("create_plan: negative stencil extents");
    if (dir == SG_DIR_X && (ext.top != 0 || ext.bottom != 0))
      sg::invalid("create_plan: X-direction stencil requires top = bottom = 0");
    if (dir == SG_DIR_Y && (ext.left != 0 || ext.right != 0))
      sg::invalid("create_plan: Y-direction stencil requires left = right = 0");
    if (ext.left >= nx || ext.right >= nx || ext.top >= ny || ext.bottom >= ny)
      sg::invalid("create_plan: stencil extents must be smaller than the grid");
    const long long W = ext.left + ext.right + 1, H = ext.top + ext.bottom + 1;
    if (fn == SG_FN_NONE) {
      if (count == 0) sg::invalid("create_plan: empty weight array");
      if (static_cast<long long>(count) != W * H)
        sg::invalid("create_plan: weight count does not match the stencil window");
      for (size_t k = 0; k < count; ++k)
        if (!std::isfinite(values[k])) sg::invalid("create_plan: non-finite stencil weight");
    } else {
      int mw, mh, mc;
      if (!sg::function_shape(fn, &mw, &mh, &mc))
        sg::invalid("create_plan: null stencil function");
      // The reference would read outside the window / coefficient array
      // (undefined behaviour); the device path rejects it instead.
      if (W < mw || H < mh)
        sg::invalid(std::string("create_plan: window smaller than ") + sg::function_name(fn) + " reads");
      if (static_cast<long long>(count) < mc)
        sg::invalid(std::string("create_plan: too few coefficients for ") + sg::function_name(fn));
      if (W * H > 256 && !(W == 3 && H <= 3))
        sg::invalid("create_plan: device function windows are limited to 256 taps");
      if (fn >= SG_FN_JIT_BASE && count > 256)
        sg::invalid("create_plan: at most 256 coefficients for a source function");
    }
    if (numWorkers < 1) sg::invalid("create_plan: numWorkers must be >= 1");
    auto tiles = tiles_for(ny, numTiles);
    require_device();

    auto* p = new sg_plan_s();
    p->dir = dir;
    p->mode = mode;
    p->ext = ext;
    p->fn = fn;
    p->values.assign(values, values + count);
    p->dtype = dtype;
    p->nx = nx;
    p->ny = ny;
    p->memory = memory;
    p->numTiles = numTiles;
    p->numWorkers = numWorkers;
    p->tiles = std::move(tiles);
    try {
      SG_CUDA(cudaGetDevice(&p->device));
      // a BLOCKING stream: ordered after work the caller queued on the legacy
      // default stream (e.g. torch kernels producing device inputs)
      SG_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamDefault));
      // numWorkers -> GPUs for host grids (device grids live on one device)
      int ndev = 1;
      SG_CUDA(cudaGetDeviceCount(&ndev));
      int G = device_map() == 1 ? numWorkers : std::min(numWorkers, ndev);
      G = std::min(G, ny);
      if (memory == SG_MEM_HOST && G > 1) setup_workers(p, G, ndev);
      if (memory == SG_MEM_HOST && p->workers.empty()) {
        const char* force = std::getenv("SG_STREAM_PLANS");
        size_t freeB = 0, totalB = 0;
        SG_CUDA(cudaMemGetInfo(&freeB, &totalB));
        const bool fits = 2 * p->bytes() + (512ull << 20) < freeB;
        if ((force && force[0] == '1') || !fits) {
          setup_streaming(p);
          p->streamed = true;
        }
      }
      void* ptrs[2] = {in, out};
      for (int k = 0; k < 2; ++k) {
        auto& b = p->buf[k];
        if (memory == SG_MEM_DEVICE) {
          b.dev = ptrs[k];
          b.devValid = true;
          b.hostValid = false;
        } else {
          b.host = ptrs[k];
          if (p->workers.empty() && !p->streamed) {  // multi-worker / streamed plans hold no mirrors
            SG_CUDA(cudaMalloc(&b.dev, p->bytes()));
            b.owned = true;
          }
          // Page-lock large pageable host grids once so every transfer is a
          // full-speed DMA (the plan never owns the grids; unregistered at
          // destroy). Failure to register is harmless (pageable copies).
          if (p->bytes() >= (4u << 20)) {
            cudaPointerAttributes attr{};
            if (cudaPointerGetAttributes(&attr, b.host) == cudaSuccess &&
                attr.type == cudaMemoryTypeUnregistered) {
              if (cudaHostRegister(b.host, p->bytes(), cudaHostRegisterPortable) == cudaSuccess)
                p->registered[k] = true;
              else
                cudaGetLastError();
            } else {
              cudaGetLastError();
            }
          }
        }
      }
      p->valid = true;
    } catch (...) {
      p->valid = true;
      p->release();
      delete p;
      throw;
    }
    *plan = p;
  });
}

static sg_slab_desc full_grid_desc(const sg_plan_s* p) {
  // make_geom, stencil.cpp:26-40
  sg_slab_desc d{};
  d.nx = p->nx;
  d.inRows = p->ny;
  d.inShift = 0;
  const bool periodic = p->mode == SG_PERIODIC;
  d.wrapX = d.wrapY = periodic ? 1 : 0;
  d.row0 = periodic ? 0 : p->ext.top;
  d.row1 = periodic ? p->ny : p->ny - p->ext.bottom;
  if (periodic) {
    d.col0 = 0;
    d.col1 = p->nx;
  } else {
    const int fastLo = std::min(p->ext.left, p->nx);
    const int hi = std::min(p->nx - p->ext.right, p->nx);
    d.col0 = fastLo;
    d.col1 = std::max(hi, fastLo);
  }
  return d;
}

// Streamed host plan: rows [a, b) of the computed range per chunk. The
// input slot holds global rows a - top .. b + bottom - 1 (wrapped modulo ny
// when periodic; a non-periodic range never leaves the grid), the kernel
// computes the chunk's rows into the output slot (the same slab launch the
// multi-GPU path uses: inShift = top, no y wrap), and the output rows go
// back — only the computed columns of a non-periodic grid, so the host
// frame stays untouched (stencil.cpp:35-38). H2D, kernels and D2H run on
// three streams over a ring of NSLOT slots.
static void streamed_host_compute(sg_plan_s* p, sg_plan_s::Buf& in, sg_plan_s::Buf& out, cudaStream_t s) {
  const int ny = p->ny, top = p->ext.top, bottom = p->ext.bottom, R = p->chunkRows;
  const size_t eb = p->elem(), rowB = static_cast<size_t>(p->nx) * eb;
  if (!p->sH2D) SG_CUDA(cudaStreamCreateWithFlags(&p->sH2D, cudaStreamNonBlocking));
  if (!p->sD2H) SG_CUDA(cudaStreamCreateWithFlags(&p->sD2H, cudaStreamNonBlocking));
  const sg_slab_desc g = full_grid_desc(p);
  const bool periodic = p->mode == SG_PERIODIC;
  cudaEvent_t start = nullptr;
  if (p->events.empty()) {
    p->events.resize(1);
    SG_CUDA(cudaEventCreateWithFlags(&p->events[0], cudaEventDisableTiming));
  }
  start = p->events[0];
  SG_CUDA(cudaEventRecord(start, s));
  SG_CUDA(cudaStreamWaitEvent(p->sH2D, start, 0));
  SG_CUDA(cudaStreamWaitEvent(p->sD2H, start, 0));
  const auto* hin = static_cast<const char*>(in.host);
  auto* hout = static_cast<char*>(out.host);
  int k = 0;
  for (int a = g.row0; a < g.row1; a += R, ++k) {
    const int b = std::min(a + R, g.row1);
    auto& sl = p->slots[k % sg_plan_s::NSLOT];
    // the slot's previous chunk: its kernel has read `in`, its D2H has read `out`
    if (sl.used) {
      SG_CUDA(cudaStreamWaitEvent(p->sH2D, sl.computed, 0));
    }
    // input rows a - top .. b + bottom - 1, split where they wrap
    char* din = static_cast<char*>(sl.in);
    int row = a - top, dst = 0;
    const int last = b + bottom;
    while (row < last) {
      const int gr = periodic ? ((row % ny) + ny) % ny : row;
      const int n = std::min(last - row, ny - gr);
      SG_CUDA(cudaMemcpyAsync(din + static_cast<size_t>(dst) * rowB, hin + static_cast<size_t>(gr) * rowB,
                              static_cast<size_t>(n) * rowB, cudaMemcpyHostToDevice, p->sH2D));
      row += n;
      dst += n;
    }
    SG_CUDA(cudaEventRecord(sl.loaded, p->sH2D));
    SG_CUDA(cudaStreamWaitEvent(s, sl.loaded, 0));
    if (sl.used) SG_CUDA(cudaStreamWaitEvent(s, sl.drained, 0));
    sg_slab_desc d = g;
    d.inRows = (b - a) + top + bottom;
    d.inShift = top;
    d.row0 = 0;
    d.row1 = b - a;
    d.wrapY = 0;
    sg::launch_stencil(d, p->ext, p->fn, p->values.data(), p->values.size(), p->dtype, sl.in, sl.out, s);
    SG_CUDA(cudaEventRecord(sl.computed, s));
    SG_CUDA(cudaStreamWaitEvent(p->sD2H, sl.computed, 0));
    const size_t c0 = static_cast<size_t>(g.col0) * eb, w = static_cast<size_t>(g.col1 - g.col0) * eb;
    if (w > 0)
      SG_CUDA(cudaMemcpy2DAsync(hout + static_cast<size_t>(a) * rowB + c0, rowB, static_cast<char*>(sl.out) + c0,
                                rowB, w, static_cast<size_t>(b - a), cudaMemcpyDeviceToHost, p->sD2H));
    SG_CUDA(cudaEventRecord(sl.drained, p->sD2H));
    sl.used = true;
  }
  SG_CUDA(cudaStreamSynchronize(p->sD2H));
  SG_CUDA(cudaStreamSynchronize(s));
  for (auto& sl : p->slots) sl.used = false;
}

// Residency::Host on a large periodic grid: stream the grid through the GPU
// in row chunks on three streams so the H2D of chunk k+1, the kernel on
// chunk k and the D2H of chunk k-1 overlap (PCIe is full duplex). Each
// chunk's kernel waits only for the chunks holding its halo rows.
static void pipelined_host_compute(sg_plan_s* p, sg_plan_s::Buf& in, sg_plan_s::Buf& out, cudaStream_t s) {
  const int ny = p->ny, top = p->ext.top, bottom = p->ext.bottom;
  const size_t rowBytes = static_cast<size_t>(p->nx) * p->elem();
  // chunk count: the pipeline's fill (first H2D) and drain (last D2H) cost
  // one chunk each. Config 4 e2e: 32 chunks 5.77, 64 5.87, 128 5.99, 256
  // 5.90 Gpts/s. SG_PIPE_CHUNKS overrides (A/B).
  static const int chunks = [] {
    const char* e = std::getenv("SG_PIPE_CHUNKS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 128;
  }();
  int rows = std::max((ny + chunks - 1) / chunks, std::max(std::max(top, bottom), 1));
  const int nch = (ny + rows - 1) / rows;
  if (!p->sH2D) SG_CUDA(cudaStreamCreateWithFlags(&p->sH2D, cudaStreamNonBlocking));
  if (!p->sD2H) SG_CUDA(cudaStreamCreateWithFlags(&p->sD2H, cudaStreamNonBlocking));
  const size_t need = 2 * static_cast<size_t>(nch) + 2;
  while (p->events.size() < need) {
    cudaEvent_t e;
    SG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->events.push_back(e);
  }
  cudaEvent_t evStart = p->events[0], evEnd = p->events[1];
  cudaEvent_t* evH2D = p->events.data() + 2;
  cudaEvent_t* evComp = p->events.data() + 2 + nch;
  auto* hin = static_cast<const char*>(in.host);
  auto* din = static_cast<char*>(in.dev);
  SG_CUDA(cudaEventRecord(evStart, s));
  SG_CUDA(cudaStreamWaitEvent(p->sH2D, evStart, 0));
  SG_CUDA(cudaStreamWaitEvent(p->sD2H, evStart, 0));
  if (top > 0) {  // wrapped halo of chunk 0: the last `top` rows
    const size_t off = static_cast<size_t>(ny - top) * rowBytes;
    SG_CUDA(cudaMemcpyAsync(din + off, hin + off, top * rowBytes, cudaMemcpyHostToDevice, p->sH2D));
  }
  for (int k = 0; k < nch; ++k) {
    // rows [ny - top, ny) went up first (chunk 0's wrapped halo) and chunk
    // 0's kernel may be reading them: never write them again
    const int a = k * rows, b = std::min(std::min(ny, a + rows), ny - top);
    const size_t off = static_cast<size_t>(a) * rowBytes;
    if (b > a) SG_CUDA(cudaMemcpyAsync(din + off, hin + off, (b - a) * rowBytes, cudaMemcpyHostToDevice, p->sH2D));
    SG_CUDA(cudaEventRecord(evH2D[k], p->sH2D));
  }
  sg_slab_desc d = full_grid_desc(p);
  for (int k = 0; k < nch; ++k) {
    const int a = k * rows, b = std::min(ny, a + rows);
    // rows up to b-1+bottom must be resident (wrapping to chunk 0 is covered
    // by stream order: chunk 0 was uploaded before every later chunk)
    const int lastRow = std::min(ny - 1, b - 1 + bottom);
    SG_CUDA(cudaStreamWaitEvent(s, evH2D[lastRow / rows], 0));
    d.row0 = a;
    d.row1 = b;
    sg::launch_stencil(d, p->ext, p->fn, p->values.data(), p->values.size(), p->dtype, in.dev, out.dev, s);
    SG_CUDA(cudaEventRecord(evComp[k], s));
    SG_CUDA(cudaStreamWaitEvent(p->sD2H, evComp[k], 0));
    const size_t off = static_cast<size_t>(a) * rowBytes;
    SG_CUDA(cudaMemcpyAsync(static_cast<char*>(out.host) + off, static_cast<const char*>(out.dev) + off,
                            (b - a) * rowBytes, cudaMemcpyDeviceToHost, p->sD2H));
  }
  SG_CUDA(cudaEventRecord(evEnd, p->sD2H));
  SG_CUDA(cudaStreamWaitEvent(s, evEnd, 0));
}

}  // extern "C"

// ---------------------------------------------- multi-worker (multi-GPU)

static void setup_workers(sg_plan_s* p, int G, int ndev) {
  const auto t = tiles_for(p->ny, G);  // make_tiles' ceil-first row blocks
  const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
  const int H = p->ext.top + p->ext.bottom;
  p->workers.resize(G);
  for (int w = 0; w < G; ++w) {
    auto& W = p->workers[w];
    W.device = w % ndev;
    W.r0 = t[w].first;
    W.r1 = t[w].second;
    SG_CUDA(cudaSetDevice(W.device));
    SG_CUDA(cudaStreamCreateWithFlags(&W.stream, cudaStreamNonBlocking));
    SG_CUDA(cudaEventCreateWithFlags(&W.done, cudaEventDisableTiming));
    for (int k = 0; k < 2; ++k) SG_CUDA(cudaMalloc(&W.buf[k], (W.own() + H) * rowB));
  }
  // peer access between the devices in use (halo refreshes go over NVLink;
  // without it cudaMemcpyPeerAsync stages through the host)
  const int used = std::min(G, ndev);
  for (int a = 0; a < used; ++a)
    for (int b = 0; b < used; ++b) {
      int can = 0;
      if (a == b || cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) continue;
      cudaSetDevice(a);
      if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
    }
  SG_CUDA(cudaSetDevice(p->device));
}

// Slab launch descriptor of worker W: output rows in slab-local coordinates
// (make_geom, stencil.cpp:26-40, restricted to the worker's rows).
static sg_slab_desc worker_desc(const sg_plan_s* p, const sg_plan_s::Worker& W) {
  sg_slab_desc d = full_grid_desc(p);
  d.inRows = W.own() + p->ext.top + p->ext.bottom;
  d.inShift = p->ext.top;
  d.wrapY = 0;  // halos are explicit rows of the slab
  const int g0 = std::max(W.r0, d.row0), g1 = std::min(W.r1, d.row1);
  d.row0 = g0 - W.r0;
  d.row1 = std::max(g1, g0) - W.r0;
  return d;
}

// Global row held by ext row k of worker W (-1: outside a non-periodic grid).
static int ext_global_row(const sg_plan_s* p, const sg_plan_s::Worker& W, int k) {
  const int g = W.r0 - p->ext.top + k;
  if (p->mode == SG_PERIODIC) return ((g % p->ny) + p->ny) % p->ny;
  return g >= 0 && g < p->ny ? g : -1;
}

// H2D of ext rows [k0, k1) of worker W's slab `dst` from the host grid, as
// contiguous runs of global rows (the periodic wrap splits a run).
static void upload_ext_rows(const sg_plan_s* p, const sg_plan_s::Worker& W, const void* host, void* dst, int k0,
                            int k1, cudaStream_t s) {
  const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
  int k = k0;
  while (k < k1) {
    const int g = ext_global_row(p, W, k);
    if (g < 0) {
      ++k;
      continue;
    }
    int len = 1;
    while (k + len < k1 && ext_global_row(p, W, k + len) == g + len) ++len;
    SG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + k * rowB, static_cast<const char*>(host) + g * rowB,
                            len * rowB, cudaMemcpyHostToDevice, s));
    k += len;
  }
}

// Device-resident input: refresh every worker's halo rows of binding `k`
// from the workers that own those rows (peer copies), after joining every
// worker's previous work.
static void refresh_halos(sg_plan_s* p, int k) {
  const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
  const int top = p->ext.top, H = top + p->ext.bottom;
  if (H == 0) return;
  std::vector<int> owner(p->ny);
  for (size_t u = 0; u < p->workers.size(); ++u)
    for (int g = p->workers[u].r0; g < p->workers[u].r1; ++g) owner[g] = static_cast<int>(u);
  for (auto& W : p->workers) {
    SG_CUDA(cudaSetDevice(W.device));
    for (auto& U : p->workers) SG_CUDA(cudaStreamWaitEvent(W.stream, U.done, 0));
    for (int e = 0; e < W.own() + H; ++e) {
      if (e >= top && e < top + W.own()) continue;  // own rows
      const int g = ext_global_row(p, W, e);
      if (g < 0) continue;
      const auto& U = p->workers[owner[g]];
      const char* src = static_cast<const char*>(U.buf[k]) + (top + g - U.r0) * rowB;
      char* dst = static_cast<char*>(W.buf[k]) + e * rowB;
      SG_CUDA(cudaMemcpyPeerAsync(dst, W.device, src, U.device, rowB, W.stream));
    }
    SG_CUDA(cudaEventRecord(W.done, W.stream));
  }
}

// compute() of a multi-worker plan: every worker runs the stencil on its
// slab on its own device and stream; the result is bitwise the single-GPU
// one (same kernel arithmetic per point).
static void compute_workers(sg_plan_s* p, sg_residency residency, cudaStream_t caller, int synchronize) {
  const int ii = p->inIdx, oi = 1 - p->inIdx;
  auto& in = p->buf[ii];
  auto& out = p->buf[oi];
  const bool periodic = p->mode == SG_PERIODIC;
  const int top = p->ext.top, H = top + p->ext.bottom;
  const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
  const bool uploadIn = !in.devValid || (residency == SG_RESIDENCY_HOST && in.hostValid);
  if (uploadIn && !in.hostValid) sg::logic("compute: input has no valid copy");
  // the frame of a non-periodic output keeps the caller's values
  const bool uploadOut = !periodic && out.hostValid && (!out.devValid || residency == SG_RESIDENCY_HOST);
  const bool download = residency == SG_RESIDENCY_HOST;
  // order after the caller's stream (an event of the caller's device: the
  // current device here; destruction is deferred until it completes)
  int callerDev = p->device;
  SG_CUDA(cudaGetDevice(&callerDev));
  cudaEvent_t start;
  SG_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  SG_CUDA(cudaEventRecord(start, caller));
  if (!uploadIn && !in.halosValid) refresh_halos(p, ii);
  // row-chunk pipeline on large grids: ~128 chunks over the whole grid
  const int totalChunks = p->bytes() >= (64u << 20) ? 128 : 1;
  const int G = static_cast<int>(p->workers.size());
  for (auto& W : p->workers) {
    SG_CUDA(cudaSetDevice(W.device));
    SG_CUDA(cudaStreamWaitEvent(W.stream, start, 0));
    for (auto& U : p->workers) SG_CUDA(cudaStreamWaitEvent(W.stream, U.done, 0));
    const sg_slab_desc d0 = worker_desc(p, W);
    char* din = static_cast<char*>(W.buf[ii]);
    char* dout = static_cast<char*>(W.buf[oi]);
    if (uploadOut)
      SG_CUDA(cudaMemcpyAsync(dout + top * rowB, static_cast<const char*>(out.host) + W.r0 * rowB,
                              W.own() * rowB, cudaMemcpyHostToDevice, W.stream));
    const int outRows = d0.row1 - d0.row0;
    int nch = uploadIn ? std::max(1, std::min(outRows, (totalChunks + G - 1) / G)) : 1;
    if (nch > 1) {
      if (!W.sH2D) SG_CUDA(cudaStreamCreateWithFlags(&W.sH2D, cudaStreamNonBlocking));
      if (!W.sD2H) SG_CUDA(cudaStreamCreateWithFlags(&W.sD2H, cudaStreamNonBlocking));
      while (W.ev.size() < 2 * static_cast<size_t>(nch) + 1) {
        cudaEvent_t e;
        SG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        W.ev.push_back(e);
      }
      cudaEvent_t* evUp = W.ev.data();
      cudaEvent_t* evK = W.ev.data() + nch;
      cudaEvent_t evGo = W.ev[2 * nch];
      SG_CUDA(cudaEventRecord(evGo, W.stream));
      SG_CUDA(cudaStreamWaitEvent(W.sH2D, evGo, 0));
      SG_CUDA(cudaStreamWaitEvent(W.sD2H, evGo, 0));
      int up = 0;  // ext rows uploaded so far
      for (int c = 0; c < nch; ++c) {
        const int a = d0.row0 + outRows * c / nch, b = d0.row0 + outRows * (c + 1) / nch;
        // output row j reads ext rows j .. j + H
        const int need = c == nch - 1 ? W.own() + H : b + H;
        if (c == 0) up = 0;
        if (need > up) upload_ext_rows(p, W, in.host, din, up, need, W.sH2D);
        up = std::max(up, need);
        SG_CUDA(cudaEventRecord(evUp[c], W.sH2D));
        SG_CUDA(cudaStreamWaitEvent(W.stream, evUp[c], 0));
        sg_slab_desc d = d0;
        d.row0 = a;
        d.row1 = b;
        if (a < b) sg::launch_stencil(d, p->ext, p->fn, p->values.data(), p->values.size(), p->dtype, din,
                                      dout + top * rowB, W.stream);
        SG_CUDA(cudaEventRecord(evK[c], W.stream));
        if (download && a < b) {
          SG_CUDA(cudaStreamWaitEvent(W.sD2H, evK[c], 0));
          SG_CUDA(cudaMemcpyAsync(static_cast<char*>(out.host) + (W.r0 + a) * rowB, dout + (top + a) * rowB,
                                  (b - a) * rowB, cudaMemcpyDeviceToHost, W.sD2H));
        }
      }
      SG_CUDA(cudaEventRecord(evK[0], W.sD2H));  // reuse: the D2H tail
      SG_CUDA(cudaStreamWaitEvent(W.stream, evK[0], 0));
      // rows outside [row0, row1) (the non-periodic frame rows) go back as
      // uploaded: the whole own block is host-coherent
      if (download && d0.row0 > 0)
        SG_CUDA(cudaMemcpyAsync(static_cast<char*>(out.host) + W.r0 * rowB, dout + top * rowB,
                                d0.row0 * rowB, cudaMemcpyDeviceToHost, W.stream));
      if (download && d0.row1 < W.own())
        SG_CUDA(cudaMemcpyAsync(static_cast<char*>(out.host) + (W.r0 + d0.row1) * rowB,
                                dout + (top + d0.row1) * rowB, (W.own() - d0.row1) * rowB,
                                cudaMemcpyDeviceToHost, W.stream));
    } else {
      if (uploadIn) upload_ext_rows(p, W, in.host, din, 0, W.own() + H, W.stream);
      if (d0.row0 < d0.row1)
        sg::launch_stencil(d0, p->ext, p->fn, p->values.data(), p->values.size(), p->dtype, din, dout + top * rowB,
                           W.stream);
      if (download)
        SG_CUDA(cudaMemcpyAsync(static_cast<char*>(out.host) + W.r0 * rowB, dout + top * rowB, W.own() * rowB,
                                cudaMemcpyDeviceToHost, W.stream));
    }
    SG_CUDA(cudaEventRecord(W.done, W.stream));
  }
  SG_CUDA(cudaSetDevice(callerDev));
  SG_CUDA(cudaEventDestroy(start));
  for (auto& W : p->workers) SG_CUDA(cudaStreamWaitEvent(caller, W.done, 0));
  if (uploadIn) {
    in.devValid = true;
    in.halosValid = true;
  } else {
    in.halosValid = true;
  }
  out.devValid = true;
  out.halosValid = false;
  out.hostValid = download;
  if (download || synchronize)
    for (auto& W : p->workers) {
      SG_CUDA(cudaSetDevice(W.device));
      SG_CUDA(cudaStreamSynchronize(W.stream));
    }
  SG_CUDA(cudaSetDevice(p->device));
}

extern "C" {

sg_status sg_plan_compute(sg_plan_t p, sg_residency residency, void* stream, int synchronize) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("compute: plan was destroyed");
    SG_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
    if (!p->workers.empty()) {
      int sdev = p->device;
      if (stream && cudaStreamGetDevice(s, &sdev) == cudaSuccess && sdev != p->device)
        SG_CUDA(cudaSetDevice(sdev));
      compute_workers(p, residency, s, synchronize);
      return;
    }
    auto& in = p->buf[p->inIdx];
    auto& out = p->buf[1 - p->inIdx];
    if (p->streamed) {  // always host-coherent and synchronous (no device mirrors)
      if (in.host == out.host) sg::invalid("compute: bound grids alias");
      streamed_host_compute(p, in, out, s);
      return;
    }
    if (in.dev == out.dev) sg::invalid("compute: bound grids alias");
    const bool periodic = p->mode == SG_PERIODIC;
    if (p->memory == SG_MEM_HOST && !periodic && residency == SG_RESIDENCY_HOST && in.hostValid &&
        out.hostValid && p->bytes() >= (64u << 20)) {
      // a large non-periodic host compute: the streamed pipeline (its frame
      // handling downloads only the computed columns); the mirrors go stale
      if (!p->slots[0].in) setup_streaming(p);
      streamed_host_compute(p, in, out, s);
      in.devValid = false;
      out.devValid = false;
      return;
    }
    if (p->memory == SG_MEM_HOST && periodic && residency == SG_RESIDENCY_HOST && in.hostValid &&
        p->bytes() >= (64u << 20)) {
      pipelined_host_compute(p, in, out, s);
      in.devValid = true;
      out.devValid = true;
      out.hostValid = true;
      SG_CUDA(cudaStreamSynchronize(s));
      return;
    }
    if (p->memory == SG_MEM_HOST) {
      // HOST residency: a host grid holding valid values is authoritative
      // (re-uploaded on every compute); a grid whose newest values were left
      // on the device by a Device-residency compute is used from there.
      if (!in.devValid || (residency == SG_RESIDENCY_HOST && in.hostValid)) {
        if (!in.hostValid) sg::logic("compute: input has no valid copy");
        SG_CUDA(cudaMemcpyAsync(in.dev, in.host, p->bytes(), cudaMemcpyHostToDevice, s));
        in.devValid = true;
      }
      // Non-periodic stencils leave the output frame untouched: the device
      // output must carry the caller's frame values.
      if (!periodic && (!out.devValid || (residency == SG_RESIDENCY_HOST && out.hostValid))) {
        SG_CUDA(cudaMemcpyAsync(out.dev, out.host, p->bytes(), cudaMemcpyHostToDevice, s));
        out.devValid = true;
      }
    }
    const sg_slab_desc d = full_grid_desc(p);
    sg::launch_stencil(d, p->ext, p->fn, p->values.data(), p->values.size(), p->dtype, in.dev,
                       out.dev, s);
    out.devValid = true;
    if (p->memory == SG_MEM_HOST) {
      out.hostValid = false;
      if (residency == SG_RESIDENCY_HOST) {
        SG_CUDA(cudaMemcpyAsync(out.host, out.dev, p->bytes(), cudaMemcpyDeviceToHost, s));
        out.hostValid = true;
        synchronize = 1;  // host result must be complete on return
      }
    }
    if (synchronize) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_plan_swap(sg_plan_t p) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("swap_plan: plan was destroyed");
    p->inIdx = 1 - p->inIdx;
  });
}

sg_status sg_plan_destroy(sg_plan_t* p) {
  return guard([&] {
    if (!p || !*p) return;
    (*p)->release();
    delete *p;
    *p = nullptr;
  });
}

sg_status sg_plan_sync_to_host(sg_plan_t p) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("sync_to_host: plan was destroyed");
    if (p->memory != SG_MEM_HOST) return;
    if (!p->workers.empty()) {
      const size_t rowB = static_cast<size_t>(p->nx) * p->elem();
      for (int k = 0; k < 2; ++k) {
        auto& b = p->buf[k];
        if (b.hostValid || !b.devValid) continue;
        for (auto& W : p->workers) {
          SG_CUDA(cudaSetDevice(W.device));
          SG_CUDA(cudaMemcpyAsync(static_cast<char*>(b.host) + W.r0 * rowB,
                                  static_cast<const char*>(W.buf[k]) + p->ext.top * rowB, W.own() * rowB,
                                  cudaMemcpyDeviceToHost, W.stream));
        }
        b.hostValid = true;
      }
      for (auto& W : p->workers) {
        SG_CUDA(cudaSetDevice(W.device));
        SG_CUDA(cudaStreamSynchronize(W.stream));
      }
      SG_CUDA(cudaSetDevice(p->device));
      return;
    }
    SG_CUDA(cudaSetDevice(p->device));
    for (auto& b : p->buf)
      if (!b.hostValid && b.devValid) {
        SG_CUDA(cudaMemcpyAsync(b.host, b.dev, p->bytes(), cudaMemcpyDeviceToHost, p->stream));
        b.hostValid = true;
      }
    SG_CUDA(cudaStreamSynchronize(p->stream));
  });
}

sg_status sg_plan_mark_host_dirty(sg_plan_t p, int which) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("mark_host_dirty: plan was destroyed");
    if (which != 0 && which != 1) sg::invalid("mark_host_dirty: which must be 0 or 1");
    auto& b = p->buf[which == 0 ? p->inIdx : 1 - p->inIdx];
    if (p->memory == SG_MEM_HOST) {
      b.hostValid = true;
      b.devValid = false;
    }
  });
}

sg_status sg_plan_binding(sg_plan_t p, int which, void** host_ptr, void** device_ptr) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("binding: plan was destroyed");
    if (which != 0 && which != 1) sg::invalid("binding: which must be 0 or 1");
    auto& b = p->buf[which == 0 ? p->inIdx : 1 - p->inIdx];
    if (host_ptr) *host_ptr = b.host;
    if (device_ptr) *device_ptr = b.dev;
  });
}

int sg_plan_valid(sg_plan_t p) { return p && p->valid ? 1 : 0; }

sg_status sg_set_device_map(int mode) {
  return guard([&] {
    if (mode != 0 && mode != 1) sg::invalid("set_device_map: mode must be 0 (clip) or 1 (modulo)");
    g_device_map.store(mode);
  });
}

int sg_get_device_map(void) { return device_map(); }

sg_status sg_plan_workers(sg_plan_t p, int* workers, int* devices, int* rowBegins, int* rowEnds, int capacity) {
  return guard([&] {
    if (!p || !p->valid) sg::logic("plan_workers: plan was destroyed");
    const int G = p->workers.empty() ? 1 : static_cast<int>(p->workers.size());
    if (workers) *workers = G;
    for (int w = 0; w < G && w < capacity; ++w) {
      const bool multi = !p->workers.empty();
      if (devices) devices[w] = multi ? p->workers[w].device : p->device;
      if (rowBegins) rowBegins[w] = multi ? p->workers[w].r0 : 0;
      if (rowEnds) rowEnds[w] = multi ? p->workers[w].r1 : p->ny;
    }
  });
}

int sg_plan_kernel_kind(sg_plan_t p) {
  if (!p || !p->valid) return -1;
  if (!p->workers.empty()) {
    const auto& W = p->workers[0];
    const size_t off = static_cast<size_t>(p->ext.top) * p->nx * p->elem();
    return sg::stencil_kernel_kind(worker_desc(p, W), p->ext, p->fn, p->values.size(), p->dtype,
                                   W.buf[p->inIdx], static_cast<char*>(W.buf[1 - p->inIdx]) + off);
  }
  sg_slab_desc d = full_grid_desc(p);
  if (p->streamed) {
    d.inRows = p->chunkRows + p->ext.top + p->ext.bottom;
    d.inShift = p->ext.top;
    d.row0 = 0;
    d.row1 = p->chunkRows;
    d.wrapY = 0;
    return sg::stencil_kernel_kind(d, p->ext, p->fn, p->values.size(), p->dtype, p->slots[0].in, p->slots[0].out);
  }
  return sg::stencil_kernel_kind(d, p->ext, p->fn, p->values.size(), p->dtype,
                                 p->buf[p->inIdx].dev, p->buf[1 - p->inIdx].dev);
}

sg_status sg_weno_advect(const double* phi, const double* u, const double* v, int nx, int ny, double dx,
                         double dy, double* out, sg_memory memory, void* stream) {
  return guard([&] {
    // weno.cpp:51-53
    if (nx < 7 || ny < 7) sg::invalid("weno_advect: need nx, ny >= 7");
    if (!(dx > 0.0) || !(dy > 0.0)) sg::invalid("weno_advect: dx and dy must be > 0");
    require_device();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = sizeof(double) * static_cast<size_t>(nx) * ny;
    if (memory == SG_MEM_DEVICE) {
      sg::launch_weno(phi, u, v, out, nx, ny, dx, dy, s);
      if (!stream) SG_CUDA(cudaStreamSynchronize(s));
      return;
    }
    double* d = nullptr;
    sg::retain_async_pool();
    SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 4 * bytes, s));
    double* dp = d;
    double* du = d + static_cast<size_t>(nx) * ny;
    double* dv = du + static_cast<size_t>(nx) * ny;
    double* dout = dv + static_cast<size_t>(nx) * ny;
    SG_CUDA(cudaMemcpyAsync(dp, phi, bytes, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(du, u, bytes, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(dv, v, bytes, cudaMemcpyHostToDevice, s));
    sg::launch_weno(dp, du, dv, dout, nx, ny, dx, dy, s);
    SG_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaFreeAsync(d, s));
    SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_stencil_launch(const sg_slab_desc* desc, sg_extents ext, sg_function fn,
                            const double* values, size_t count, sg_dtype dtype, const void* in,
                            void* out, void* stream) {
  return guard([&] {
    if (!desc) sg::invalid("stencil_launch: null descriptor");
    const sg_slab_desc& d = *desc;
    if (d.nx < 1 || d.inRows < 1) sg::invalid("stencil_launch: empty input");
    if (d.col0 < 0 || d.col1 > d.nx || d.row0 < 0) sg::invalid("stencil_launch: bad output window");
    if (!d.wrapY && d.row1 > d.row0 &&
        (d.row0 + d.inShift - ext.top < 0 || d.row1 - 1 + d.inShift + ext.bottom >= d.inRows))
      sg::invalid("stencil_launch: rows outside the input slab (missing halo)");
    if (in == out) sg::invalid("stencil_launch: input and output must be distinct buffers");
    require_device();
    sg::launch_stencil(d, ext, fn, values, count, dtype, in, out, static_cast<cudaStream_t>(stream));
  });
}

sg_status sg_stencil_launch_p2p(const sg_slab_desc* desc, sg_extents ext, sg_function fn, const double* values,
                                size_t count, sg_dtype dtype, const void* in, void* out, void* peerUp, int upRows,
                                void* peerDn, int dnRow0, void* stream) {
  return guard([&] {
    if (!desc) sg::invalid("stencil_launch: null descriptor");
    const sg_slab_desc& d = *desc;
    if (d.nx < 1 || d.inRows < 1) sg::invalid("stencil_launch: empty input");
    if (d.col0 < 0 || d.col1 > d.nx || d.row0 < 0) sg::invalid("stencil_launch: bad output window");
    if (!d.wrapY && d.row1 > d.row0 &&
        (d.row0 + d.inShift - ext.top < 0 || d.row1 - 1 + d.inShift + ext.bottom >= d.inRows))
      sg::invalid("stencil_launch: rows outside the input slab (missing halo)");
    if (in == out) sg::invalid("stencil_launch: input and output must be distinct buffers");
    if (upRows < 0 || dnRow0 < 0) sg::invalid("stencil_launch: bad P2P row range");
    require_device();
    sg::PeerRows pr;
    pr.up = peerUp;
    pr.dn = peerDn;
    pr.upRows = upRows;
    pr.dnRow0 = dnRow0;
    sg::launch_stencil(d, ext, fn, values, count, dtype, in, out, static_cast<cudaStream_t>(stream), pr);
  });
}

}  // extern "C"
