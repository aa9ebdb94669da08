// C-ABI glue: error reporting, device queries, host helpers (numpy pairwise
// plan, OpenBLAS order dispatch) and the attention dispatcher.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "tc_common.cuh"

namespace {
thread_local std::string g_last_error;
}

namespace ac_host {
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
int check_cuda(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return AC_ERR_CUDA;
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_attr_done;  // (kernel, device) -> bytes set
std::mutex g_sm_mu;
int g_sms[64] = {0};
}  // namespace

int func_smem(const void* fn, int bytes, const char* what) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return check_cuda(e, what);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_attr_done.find({fn, dev});
  if (it != g_attr_done.end() && it->second >= bytes) return AC_OK;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return check_cuda(e, what);
  g_attr_done[{fn, dev}] = bytes;
  return AC_OK;
}

// per calling thread, like the assign/update modes (a CUDA graph keeps the
// attribute its kernels were captured with); env AC_PDL sets the default
static int pdl_default() { return getenv("AC_PDL") ? atoi(getenv("AC_PDL")) : 1; }
thread_local int g_pdl = pdl_default();
bool pdl_on() { return g_pdl != 0; }

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(g_sm_mu);
  if (!g_sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}
}  // namespace ac_host

// ---------------------------------------------------------------------------
// TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry
// point, so the library does not link libcuda directly)
// ---------------------------------------------------------------------------
namespace ac_host {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                int64_t rows, int64_t cols, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return AC_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * elem_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return AC_ERR_CUDA;
  }
  return AC_OK;
}
}  // namespace ac_host

extern "C" const char* ac_last_error(void) { return g_last_error.c_str(); }
extern "C" int ac_abi_version(void) { return AC_ABI_VERSION; }

extern "C" int ac_struct_sizes(int64_t* out3) {
  out3[0] = (int64_t)sizeof(ac_cluster_problem);
  out3[1] = (int64_t)sizeof(ac_select_problem);
  out3[2] = (int64_t)sizeof(ac_attn_item);
  return AC_OK;
}

extern "C" int ac_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return ac_host::check_cuda(e, "cudaGetDevice");
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return ac_host::check_cuda(e, "cudaGetDeviceProperties");
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return AC_OK;
}

// ---------------------------------------------------------------------------
// numpy pairwise-sum plan (layout documented in pairwise.cuh)
// ---------------------------------------------------------------------------
namespace {
struct PlanNode { int a, b, height; };
struct PlanBuilder {
  std::vector<int32_t> leaves;  // leaf start offsets (DFS order)
  std::vector<PlanNode> internal;
  std::vector<int> leaf_height;  // always 0
  // returns encoded id: >= 0 leaf index, < 0 -(internal index + 1)
  int build(int64_t lo, int64_t n, int& height) {
    if (n <= 128) {
      leaves.push_back((int32_t)lo);
      height = 0;
      return (int)leaves.size() - 1;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    int ha, hb;
    const int a = build(lo, n2, ha);
    const int b = build(lo + n2, n - n2, hb);
    height = (ha > hb ? ha : hb) + 1;
    internal.push_back({a, b, height});
    return -(int)internal.size();
  }
};
std::vector<int32_t> make_plan(int64_t n) {
  PlanBuilder pb;
  int h = 0;
  pb.build(0, n, h);
  const int L = (int)pb.leaves.size();
  const int I = (int)pb.internal.size();
  auto resolve = [&](int id) { return id >= 0 ? id : L + (-id - 1); };
  int H = 0;
  for (auto& nd : pb.internal) H = nd.height > H ? nd.height : H;
  std::vector<int32_t> plan;
  plan.push_back(L);
  plan.push_back(I);
  plan.push_back(H);
  for (int i = 0; i < L; ++i) plan.push_back(pb.leaves[i]);
  plan.push_back((int32_t)n);
  // level boundaries: internal nodes grouped by height 1..H
  std::vector<int> count(H + 2, 0);
  for (auto& nd : pb.internal) count[nd.height]++;
  int acc = 0;
  for (int hh = 1; hh <= H; ++hh) { plan.push_back(acc); acc += count[hh]; }
  plan.push_back(acc);
  for (int hh = 1; hh <= H; ++hh)
    for (int j = 0; j < I; ++j)
      if (pb.internal[j].height == hh) {
        plan.push_back(L + j);
        plan.push_back(resolve(pb.internal[j].a));
        plan.push_back(resolve(pb.internal[j].b));
      }
  return plan;
}
}  // namespace

extern "C" int64_t ac_pw_plan_len(int64_t n) {
  if (n < 0) return -1;
  return (int64_t)make_plan(n).size();
}

extern "C" int ac_pw_plan_build(int64_t n, int32_t* host_out, int64_t cap) {
  if (n < 0 || n > (int64_t)INT32_MAX) { ac_host::set_error("plan: bad n=%lld", (long long)n); return AC_ERR_PARAM; }
  std::vector<int32_t> p = make_plan(n);
  if ((int64_t)p.size() > cap) { ac_host::set_error("plan: capacity %lld < %zu", (long long)cap, p.size()); return AC_ERR_PARAM; }
  std::memcpy(host_out, p.data(), p.size() * sizeof(int32_t));
  return AC_OK;
}

// OpenBLAS 0.3.30 (SkylakeX) dispatch of the reference's f32 `a @ b.T`
// (numpy matmul -> cblas_sgemm / gemv), measured in the oracle host
// (re-probed by oracle/probe_blas.py).
// Measured rules: a unit dimension goes to sgemv; M*N <= 1200 with D >= 32
// goes to the AVX-512 small-matrix kernel (16 lane chains; elements in the
// (M%4) x (N%4) corner reduce with the halves tree); everything else is the
// general kernel's sequential chain.
extern "C" int ac_gemm_order(int64_t m, int64_t n, int64_t d) {
  if (m == 1 || n == 1) return AC_ORDER_GEMV8;
  if (m * n <= 1200 && d >= 32) return AC_ORDER_LANES16;
  return AC_ORDER_SEQ;
}

// ---------------------------------------------------------------------------
// attention dispatch: tcgen05 kernel for bf16 / D in {64,128}, CUDA cores
// otherwise (f32 inputs need f32 numerics for the 1e-4 parity bar)
// ---------------------------------------------------------------------------
extern "C" int ac_attention_item_rows(int dtype, int d) {
  return (dtype == AC_DTYPE_BF16 && (d == 64 || d == 128)) ? 256 : 128;
}

extern "C" int ac_sparse_attention(const void* q, int64_t q_rows_total, const int32_t* qidx,
                                   const void* k, const void* v, int dtype, int d, int64_t L,
                                   int heads, const ac_attn_item* items, int nitems,
                                   const int32_t* runs, float scale, void* out, int out_dtype,
                                   void* stream) {
  if (dtype == AC_DTYPE_BF16 && d == 64)
    return ac_sparse_attention_fa4(q, q_rows_total, qidx, k, v, d, L, heads, items, nitems, runs,
                                   scale, out, out_dtype, stream);
  if (dtype == AC_DTYPE_BF16 && d == 128)
    return ac_sparse_attention_fa4_d128(q, q_rows_total, qidx, k, v, d, L, heads, items, nitems, runs,
                                  scale, out, out_dtype, stream);
  return ac_sparse_attention_simt(q, qidx, k, v, dtype, d, L, items, nitems, runs, scale, out,
                                  out_dtype, stream);
}

// ---------------------------------------------------------------------------
// workspace sizing: byte size of every caller-owned buffer of one problem /
// one attention launch, so a non-Python caller can size its allocations from
// the header alone (engine.Batch allocates exactly these; tests/test_abi.py).
// ---------------------------------------------------------------------------
namespace {
int64_t put(int64_t* f, int nf, int i, int64_t v) {
  if (f && i < nf) f[i] = v;
  return v;
}
}  // namespace

extern "C" int64_t ac_workspace_bytes(int op, const int64_t* dims, int ndims, int64_t* fields,
                                      int nfields) {
  auto need = [&](int k) {
    if (!dims || ndims < k) {
      ac_host::set_error("ac_workspace_bytes: op %d needs %d dims, got %d", op, k, ndims);
      return false;
    }
    for (int i = 0; i < k; ++i)
      if (dims[i] < 0) {
        ac_host::set_error("ac_workspace_bytes: dims[%d] = %lld < 0", i, (long long)dims[i]);
        return false;
      }
    return true;
  };
  int64_t tot = 0;
  if (op == AC_WS_CLUSTER) {
    if (!need(5)) return -1;
    const int64_t n = dims[0], kcap = dims[1], d = dims[2], dtype = dims[3], mi = dims[4];
    const bool fast = (d == 64 || d == 128);
    const int64_t tiles = (n + 127) / 128;
    int i = 0;
    tot += put(fields, nfields, i++, 4 * n);                     // xx
    tot += put(fields, nfields, i++, 4 * kcap * d);              // centers
    tot += put(fields, nfields, i++, 4 * kcap);                  // cc
    tot += put(fields, nfields, i++, 4 * n);                     // labels
    tot += put(fields, nfields, i++, 4 * n);                     // best
    tot += put(fields, nfields, i++, 4 * kcap);                  // counts
    tot += put(fields, nfields, i++, 4 * n);                     // perm
    tot += put(fields, nfields, i++, 4 * (kcap + 1));            // starts
    tot += put(fields, nfields, i++, 4 * tiles * kcap);          // tile_hist
    tot += put(fields, nfields, i++, 4 * (mi > 0 ? mi : 1));     // inertia
    tot += put(fields, nfields, i++, 4 * kcap);                  // movement
    tot += put(fields, nfields, i++, 4 * 8);                     // status
    tot += put(fields, nfields, i++, 4 * ac_pw_plan_len(n));     // plan_n
    tot += put(fields, nfields, i++, 0);                         // plan_k (reserved)
    tot += put(fields, nfields, i++, 8 * n);                     // dscratch
    tot += put(fields, nfields, i++, (dtype == AC_DTYPE_F32 && fast) ? 2 * 3 * n * d : 0);  // planes
    tot += put(fields, nfields, i++, fast ? 8 * kcap * d : 0);   // csum
    tot += put(fields, nfields, i++, fast ? 4 * kcap * d : 0);   // cabs
    tot += put(fields, nfields, i++, fast ? 4 * kcap * d : 0);   // clsb
    return tot;
  }
  if (op == AC_WS_SELECT) {
    if (!need(4)) return -1;
    const int64_t gq = dims[0], c = dims[1], topk = dims[2], stride = dims[3];
    int i = 0;
    tot += put(fields, nfields, i++, 4 * gq * c);                // scores
    tot += put(fields, nfields, i++, 8 * gq * topk);             // selected
    tot += put(fields, nfields, i++, 4 * gq * stride * 2);       // runs
    tot += put(fields, nfields, i++, 4 * gq);                    // nruns
    tot += put(fields, nfields, i++, 8 * gq);                    // covered
    tot += put(fields, nfields, i++, 8);                         // density
    return tot;
  }
  if (op == AC_WS_ATTENTION) {
    if (!need(6)) return -1;
    const int64_t L = dims[0], heads = dims[1], gq_max = dims[2], d = dims[4], dtype = dims[5];
    const int64_t esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
    const int64_t qp_cap = L + 128 * gq_max;
    const int64_t item_cap = (L + 127) / 128 + gq_max;
    int i = 0;
    tot += put(fields, nfields, i++, heads * qp_cap * d * esz);              // qp
    tot += put(fields, nfields, i++, 4 * (heads * qp_cap + heads * gq_max)); // qidx (+ pad starts)
    tot += put(fields, nfields, i++, heads * item_cap * (int64_t)sizeof(ac_attn_item));  // items
    tot += put(fields, nfields, i++, heads * L * d * esz);                   // kp
    tot += put(fields, nfields, i++, heads * L * d * esz);                   // vp
    return tot;
  }
  ac_host::set_error("ac_workspace_bytes: unknown op %d", op);
  return -1;
}

extern "C" int ac_set_pdl(int on) {
  ac_host::g_pdl = on != 0;
  return AC_OK;
}
extern "C" int ac_get_pdl(void) { return ac_host::g_pdl; }
