// head.cu — S5+S6 standalone kernel: gathered LM head over the shortlist + fused log-softmax /
// top-k_t / remap (Alg. 1 lines 10-11).  Building blocks in head_impl.cuh.
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"

namespace ds {

template <typename T>
__global__ void __launch_bounds__((kMaxStages + 1) * 32, 1) head_kernel(const HeadArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const HeadSmem L = head_smem(a.stages, a.stage_bytes, a.nrows, a.d, (int)sizeof(T), a.lcap, 0);
  const HeadCtx c = head_ctx(smem, L);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) head_init_barriers(c, a.stages);
  if (a.pdl) pdl_wait();  // sel / sl_offsets / h_new come from upstream kernels
  head_segments(a, c);
  __syncthreads();
  if (warp == a.stages) {
    if (lane == 0) head_produce<T>(a, c);
  } else {
    head_load_h(a, c, (int)sizeof(T), threadIdx.x, a.stages * 32);
    named_bar_sync(1, a.stages * 32);
    head_consume<T>(a, c, warp, lane);
  }
  __syncthreads();
  if (a.pdl) pdl_launch_dependents();
  head_partials(a, c, a.stages * a.stage_bytes);
  const int j = head_ticket(a, c);
  if (j < 0) return;
  head_merge(a, c, a.stages * a.stage_bytes, nullptr, 0, j, min(a.nrows, (int)gridDim.x));
  head_merge_done(a, 0);  // leave the counters at zero for the next launch
}

// ------------------------------------------------------------------ host side

int max_smem_optin() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int x = 0;
    if (cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || x <= 0)
      x = 232448;
    v = x;
  }
  return v;
}

cudaError_t configure_max_smem(const void* fn, int* done) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (done[dev]) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin());
  if (e == cudaSuccess) done[dev] = 1;
  return e;
}

bool head_plan_ex(const ds_clusters* c, int B, int k_t, int64_t max_shortlist, int extra, int max_rows,
                  HeadPlan* p, int G) {
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const int rowbytes = c->d * esz;
  if (rowbytes > 2 * kStageTarget || (rowbytes % 16) != 0) return false;
  p->stage_rows = std::max(1, kStageTarget / rowbytes);
  p->stage_bytes = p->stage_rows * rowbytes;
  p->G = G > 0 ? G : num_sms();
  const int64_t ms = (max_shortlist > 0 && max_shortlist < c->V) ? max_shortlist : c->V;
  p->lcap = (int)((ms + p->G - 1) / p->G);
  p->rec = 2 + 2 * k_t;
  const int smax = max_smem_optin();
  const int per_row = rowbytes + p->lcap * 8 + 16;
  const int want_rows = std::min(std::min(B, kMaxGroups), max_rows);
  const int min_stages = 2;
  p->stages = 0;
  for (int st = kMaxStages; st >= min_stages; --st) {
    if (st * p->stage_bytes < merge_smem_bytes(p->G, k_t, st + 1)) break;
    const HeadSmem L0 = head_smem(st, p->stage_bytes, 0, c->d, esz, p->lcap, extra);
    const int rows = ((int)smax - (int)L0.total) / per_row;
    if (rows >= want_rows || (st == min_stages && rows >= 1)) {
      p->stages = st;
      p->rows_per_launch = std::max(1, std::min(want_rows, rows));
      break;
    }
    if (rows >= 1 && p->stages == 0 && st <= 6) {  // accept fewer rows per launch rather than a tiny ring
      p->stages = st;
      p->rows_per_launch = rows;
      break;
    }
  }
  if (p->stages == 0) return false;
  p->smem = head_smem(p->stages, p->stage_bytes, p->rows_per_launch, c->d, esz, p->lcap, extra).total;
  if (p->smem > (size_t)smax) return false;
  p->part_bytes = (size_t)p->G * p->rows_per_launch * p->rec * sizeof(float);
  p->launches = (B + p->rows_per_launch - 1) / p->rows_per_launch;
  return true;
}

bool head_plan(const ds_clusters* c, int B, int k_t, int64_t max_shortlist, HeadPlan* p) {
  return head_plan_ex(c, B, k_t, max_shortlist, 0, kMaxGroups, p);
}

void fill_head_args(HeadArgs& a, const ds_clusters* c, const HeadPlan& p, const void* h_new, int r0, int nr,
                    const int32_t* sel, const int32_t* sel_count, const int32_t* sl_offsets, int shared, int k_t,
                    int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp, float* lse,
                    float* z_out, int64_t z_stride, float* part, unsigned* counter, bool pdl) {
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  a.W = c->W_perm;
  a.perm = c->perm;
  a.offsets = c->offsets;
  const int goff = shared ? 0 : r0;
  a.sel = sel + (size_t)goff * c->M;
  a.sel_count = sel_count + goff;
  a.sl_off = sl_offsets + (size_t)goff * (c->M + 1);
  a.h = static_cast<const uint8_t*>(h_new) + (size_t)r0 * c->d * esz;
  a.M = c->M;
  a.nrows = nr;
  a.d = c->d;
  a.k_t = k_t;
  a.shared = shared;
  a.lcap = p.lcap;
  a.pdl = pdl ? 1 : 0;
  a.stages = p.stages;
  a.stage_bytes = p.stage_bytes;
  a.stage_rows = p.stage_rows;
  a.max_shortlist = (max_shortlist > 0 && max_shortlist < c->V) ? max_shortlist : c->V;
  a.top_ids = top_ids + (size_t)r0 * k_t;
  a.top_logits = top_logits + (size_t)r0 * k_t;
  a.top_logp = top_logp + (size_t)r0 * k_t;
  a.lse = lse + r0;
  a.z_out = z_out ? z_out + (size_t)r0 * z_stride : nullptr;
  a.z_stride = z_stride;
  a.part = part;
  a.counter = counter;
  a.record_out = nullptr;
}

template <typename T>
static cudaError_t launch_head_t(const HeadArgs& a, size_t smem, int G, cudaStream_t st, bool pdl) {
  static int configured[64] = {0};  // the attribute is per device
  {
    cudaError_t e = configure_max_smem(reinterpret_cast<const void*>(head_kernel<T>), configured);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3((a.stages + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, head_kernel<T>, a);
}

cudaError_t launch_head(const ds_clusters* c, const HeadPlan& p, const void* h_new, int B, const int32_t* sel,
                        const int32_t* sel_count, const int32_t* sl_offsets, int shared, int k_t,
                        int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp, float* lse,
                        float* z_out, int64_t z_stride, float* part, unsigned* counter, cudaStream_t st,
                        bool pdl, float* records) {
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  for (int r0 = 0; r0 < B; r0 += p.rows_per_launch) {
    const int nr = std::min(p.rows_per_launch, B - r0);
    HeadArgs a;
    fill_head_args(a, c, p, h_new, r0, nr, sel, sel_count, sl_offsets, shared, k_t, max_shortlist, top_ids,
                   top_logits, top_logp, lse, z_out, z_stride, part, counter, pdl && r0 == 0);
    a.record_out = records ? records + (size_t)r0 * (2 + 2 * k_t) : nullptr;
    const size_t smem = head_smem(p.stages, p.stage_bytes, nr, c->d, esz, p.lcap, 0).total;
    cudaError_t e = c->dtype == DS_BF16 ? launch_head_t<__nv_bfloat16>(a, smem, p.G, st, pdl && r0 == 0)
                                        : launch_head_t<float>(a, smem, p.G, st, pdl && r0 == 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ds
