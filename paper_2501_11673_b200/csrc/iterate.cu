// iterate.cu -- host side of the persistent Phase-2 kernel (iterate_kernel.cuh): shared-memory
// budget, choice of the compile-time instantiation, launch with thread-block clusters.
#include <cstdint>
#include <cstdlib>

#include "kpp_internal.h"

namespace kpp {
namespace {
constexpr int T2 = 512;
constexpr int NW2 = T2 / 32;
}  // namespace

int iterate_block_threads() { return T2; }

size_t iterate_smem_bytes(const IterParams& p, int C) {
  const long long s = p.s;
  const long long sp = (s + 1) & ~1LL;
  const long long sl = (s + C - 1) / C;
  long long bytes = 8 * 8;              // mbarriers
  bytes += ((C * sl + 1) & ~1LL) * 8;   // rp
  bytes += 3LL * p.slab * 8;            // x, m, w
  bytes += 2LL * sp * 8;                // r, y
  bytes += 2LL * T2 * 8;                // red
  bytes += 3LL * sp * 8;                // b_S (triple-buffered)
  bytes += 3LL * sp * 4;                // S (triple-buffered)
  bytes = (bytes + 127) & ~127LL;
  if (p.resident) bytes += (p.a_single ? 1LL : 2LL) * ((s + 3) & ~3LL) * p.sw * 8;
  if (p.m_in_smem) bytes += (p.m_in_smem == 2 ? 1LL : 2LL) * ((sl * s + 15) & ~15LL) * 8;
  if (p.ygl == 4) bytes += ((C * (s + 1) + 1) & ~1LL) * 8;      // partial y vectors
  return (size_t)bytes + 128;
}

using KernelFn = void (*)(const IterParams);

// instantiations (one translation unit per y placement, compiled in parallel)
KernelFn iterate_pick_reg_y0(int rpw, int cpl);
KernelFn iterate_pick_reg_y1(int rpw, int cpl);
KernelFn iterate_pick_reg_y4(int rpw, int cpl);
KernelFn iterate_pick_generic(int resident, int yg, int cd);
KernelFn iterate_pick_lean(const IterParams& p, int C, int rpw, int cpl);
size_t iterate_lean_smem_bytes(const IterParams& p, int C);

static bool reg_shape(const IterParams& p, int* rpw_out, int* cpl_out) {
  if (!p.resident || p.cd || NW2 * p.slab > 2 * T2) return false;
  int rpw = 2;
  while (16 * rpw < p.s) rpw *= 2;
  const int cpl = (p.slab + 31) / 32;
  if (rpw > 16 || cpl > 2) return false;
  *rpw_out = rpw;
  *cpl_out = cpl;
  return true;
}

static KernelFn pick_kernel(const IterParams& p) {
  int rpw = 0, cpl = 0;
  if (reg_shape(p, &rpw, &cpl)) {
    KernelFn f = p.ygl == 0 ? iterate_pick_reg_y0(rpw, cpl) : p.ygl == 1 ? iterate_pick_reg_y1(rpw, cpl)
               : p.ygl == 4 ? iterate_pick_reg_y4(rpw, cpl) : nullptr;
    if (f) return f;
  }
  return iterate_pick_generic(p.resident, p.ygl, p.cd);
}

// the resident passes run from a register tile (one slab buffer suffices)
bool iterate_register_tile(const IterParams& p) {
  int rpw = 0, cpl = 0;
  return reg_shape(p, &rpw, &cpl);
}

static void set_attrs(KernelFn fn, size_t smem, int C) {
  if (!fn) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

static cudaLaunchConfig_t make_cfg(int grid, int C, size_t smem, cudaStream_t stream, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T2);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// The lean instantiation (iterate_lean.cu) when the plan is one it serves (KPP_NO_LEAN=1: off).
static KernelFn pick_lean(const IterParams& p, int C) {
  static const bool off = getenv("KPP_NO_LEAN") != nullptr;
  int rpw = 0, cpl = 0;
  if (off || p.vranks > 1 || p.nranks > 1 || !reg_shape(p, &rpw, &cpl)) return nullptr;  // (no rank stage)
  return iterate_pick_lean(p, C, rpw, cpl);
}

bool iterate_uses_lean(const IterParams& p, int C) { return pick_lean(p, C) != nullptr; }

cudaError_t launch_iterate(cudaStream_t stream, const IterParams& p, int grid, int C, size_t smem) {
  if (KernelFn lf = pick_lean(p, C)) {
    const size_t ls = iterate_lean_smem_bytes(p, C);
    set_attrs(lf, ls, C);
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(grid, C, ls, stream, attr);
    return launch_coresident(cfg, attr, lf, p);
  }
  KernelFn fn = pick_kernel(p);
  set_attrs(fn, smem, C);
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = make_cfg(grid, C, smem, stream, attr);
  return launch_coresident(cfg, attr, fn, p);
}

int iterate_max_clusters(const IterParams& p, int C, size_t smem) {
  KernelFn fn = pick_kernel(p);
  set_attrs(fn, smem, C);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = make_cfg(C * 256, C, smem, nullptr, attr);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (const void*)fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace kpp
