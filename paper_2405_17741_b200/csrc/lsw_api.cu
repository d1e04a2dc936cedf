// lsw_api.cu -- the C ABI (include/lsw.h): validation, ctx state machine,
// dispatch of the K1/K2/K4 kernels, NCCL for the TP decode.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>        // types and enums only: the functions are bound at run time (Nccl below)

#include "lsw_internal.cuh"
#include "../../include/lsw_debug.h"

using namespace lsw;

namespace {

// NCCL, bound with dlopen on first use rather than linked: a process that has
// imported torch already holds torch's libnccl.so.2 (its own build, 2.28.x
// here), and a second NCCL under the same soname would be a different library
// in the same process.  RTLD_NOLOAD finds the one already loaded; otherwise
// the variant option nccl_path (the binding sets it to torch's copy), else the
// loader's search path.  lsw_nccl_version reports which one is bound.
struct Nccl {
  bool tried = false;
  void* h = nullptr;
  std::string path;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
std::mutex g_nccl_mu;
Nccl g_nccl;

const Nccl* nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  Nccl& n = g_nccl;
  if (n.tried) return n.h ? &n : nullptr;
  n.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    const char* p = lsw::opt_str("nccl_path");
    if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(dlsym(h, "ncclGetVersion"));
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  if (!n.GetVersion || !n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllReduce || !n.GetErrorString)
    return nullptr;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(n.AllReduce), &info) && info.dli_fname) n.path = info.dli_fname;
  n.h = h;
  return &n;
}

thread_local std::string g_last_error;

lsw_status fail(lsw_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

lsw_status cuda_fail(cudaError_t e, const char* what) {
  return fail(LSW_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

const char* kKindName[LSW_NKIND] = {"q", "k", "v", "o", "gate", "up", "down"};
// group -> kinds
const int kGroupKinds[LSW_NGROUP][3] = {{LSW_Q, LSW_K, LSW_V}, {LSW_O, -1, -1}, {LSW_GATE, LSW_UP, -1}, {LSW_DOWN, -1, -1}};
const int kGroupSize[LSW_NGROUP] = {3, 1, 2, 1};

constexpr int kSimtTM = 8, kSimtTN = 256;   // must match switch_simt.cu

// lsw_debug_set_option's table (process-wide; read at lsw_create)
std::mutex g_opt_mu;
std::map<std::string, std::string> g_opts;

}  // namespace

namespace lsw {
const char* opt_str(const char* key) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  auto it = g_opts.find(key);
  // the map's nodes are stable until the key is set again (not while a ctx is created)
  return it == g_opts.end() ? nullptr : it->second.c_str();
}
long opt_int(const char* key, long dflt) {
  const char* v = opt_str(key);
  return v ? strtol(v, nullptr, 10) : dflt;
}
long probe_int(const char* key) {
#ifdef LSW_TUNING
  return opt_int(key, 0);
#else
  (void)key;
  return 0;
#endif
}
}  // namespace lsw

struct lsw_ctx {
  lsw_config cfg;
  lsw_kind_desc kinds[LSW_NKIND];
  const void* router_w = nullptr;
  int device = 0;
  int num_sms = 148;
  GemvTune gemv;                        // GEMV launch plan (grid cap = num_sms unless the gemv_grid option)
  int impl = LSW_IMPL_SIMT;
  SwitchParams simt_geom{};     // tile table for the SIMT kernel
  TcPlan* tc = nullptr;
  DevState* d_state = nullptr;
  bool merged = false;
  uint64_t launches = 0;
  ncclComm_t comm = nullptr;
  int64_t xs_elems = 0, ys_elems = 0;
  int64_t x_off[LSW_NGROUP] = {}, y_off[LSW_NGROUP] = {};   // per-layer offsets
  int64_t x_per_layer = 0, y_per_layer = 0;
  bool has_pristine = false;            // lsw_attach_pristine called (RESTORE mode available)
  float* lora_u = nullptr;              // unmerged decode: LoRA-down products scratch
  bool fused_ready = false;             // fused switch + decode segment table built
  int unmerged_flags = 0;               // tuning builds only (probe unmerged_flags)
  // staging for lsw_decode_token_host
  void* st_x1 = nullptr;
  void* st_xs = nullptr;
  float* st_ys = nullptr;
  int32_t* st_idx = nullptr;
  float* st_gate = nullptr;
  cudaStream_t st_side = nullptr;       // lsw_decode_token_host: copies overlapped with the token
  PfPlan* pf = nullptr;                 // lsw_prefill_group: tensor-core plan (maps), built on first use
  float* prefill_u = nullptr;           // lsw_prefill_group: LoRA-down scratch
  int64_t prefill_u_elems = 0;
  void* prefill_z = nullptr;            // lsw_prefill_group (tc): (hi, lo) LoRA-up operand scratch
  int64_t prefill_z_elems = 0;
  std::vector<cudaEvent_t> st_ev;       // [0]: xs landed; [1 + l]: layer l's outputs final, [1 + L]: side joined
  // lsw_decode_token_host as a CUDA graph (option host_graph, default 1): one
  // per state (first token: merge; later: switch), captured on the second call
  // with the same host buffers, replayed on the caller's stream
  struct HostGraph {
    cudaGraphExec_t exec = nullptr;
    const void* key[5] = {};
    uint64_t launches = 0;
  } hgraph[2];
  cudaStream_t st_cap = nullptr;
  bool host_graph = true;
  uint64_t host_calls = 0;
};

#ifdef LSW_TUNING
namespace lsw { void gemv_set_trace(uint32_t* p); }
#endif
static size_t esize(const lsw_ctx* c) { return c->cfg.dtype == LSW_BF16 ? 2 : 4; }

static void fill_switch_params(const lsw_ctx* c, SwitchParams& p, int tm, int tn) {
  memset(&p, 0, sizeof(p));
  int64_t t = 0;
  for (int k = 0; k < LSW_NKIND; ++k) {
    KindGeom& g = p.kind[k];
    g.W = c->kinds[k].W;
    g.A = c->kinds[k].A;
    g.B = c->kinds[k].B;
    g.d_out = c->kinds[k].d_out;
    g.d_in = c->kinds[k].d_in;
    g.row_tiles = (int32_t)((g.d_out + tm - 1) / tm);
    g.col_tiles = (int32_t)((g.d_in + tn - 1) / tn);
    g.tile_begin = t;
    t += (int64_t)c->cfg.n_layers * g.row_tiles * g.col_tiles;
  }
  p.tiles_total = t;
  p.n_layers = c->cfg.n_layers;
  p.n_experts = c->cfg.n_experts;
  p.rank = c->cfg.rank;
  p.top_k = c->cfg.top_k;
  p.scale = c->cfg.alpha / (float)c->cfg.rank;
  p.state = c->d_state;
}

extern "C" {

int32_t lsw_abi_version(void) { return LSW_ABI_VERSION; }

const char* lsw_last_error(void) { return g_last_error.c_str(); }

lsw_status lsw_create(const lsw_config* cfg, const lsw_kind_desc kinds[LSW_NKIND], const void* router_w,
                      lsw_ctx** out) {
  if (!cfg || !kinds || !router_w || !out) return fail(LSW_E_ARG, "lsw_create: null argument");
  *out = nullptr;
  const lsw_config& c = *cfg;
  if (c.dtype != LSW_BF16 && c.dtype != LSW_F32) return fail(LSW_E_ARG, "lsw_create: dtype %d invalid", c.dtype);
  if (c.n_layers < 1) return fail(LSW_E_SHAPE, "lsw_create: n_layers=%d < 1", c.n_layers);
  if (c.n_experts < 1 || c.n_experts > LSW_MAX_EXPERTS)
    return fail(LSW_E_SHAPE, "lsw_create: n_experts=%d not in [1,%d]", c.n_experts, LSW_MAX_EXPERTS);
  if (c.top_k < 1 || c.top_k > c.n_experts || c.top_k > LSW_MAX_TOPK)
    return fail(LSW_E_SHAPE, "lsw_create: top_k=%d not in [1, min(n_experts=%d, %d)]", c.top_k, c.n_experts,
                LSW_MAX_TOPK);
  if (c.rank < 1 || c.rank > 64) return fail(LSW_E_SHAPE, "lsw_create: rank=%d not in [1,64]", c.rank);
  if (!(c.alpha == c.alpha) || c.alpha == 0.f) return fail(LSW_E_ARG, "lsw_create: alpha=%g invalid", c.alpha);
  if (c.d_model < 1 || c.d_model % 8) return fail(LSW_E_SHAPE, "lsw_create: d_model=%lld must be a positive multiple of 8", (long long)c.d_model);
  if (c.tp_size < 1 || c.tp_rank < 0 || c.tp_rank >= c.tp_size)
    return fail(LSW_E_ARG, "lsw_create: tp_rank=%d tp_size=%d invalid", c.tp_rank, c.tp_size);
  if (c.impl < LSW_IMPL_AUTO || c.impl > LSW_IMPL_TC) return fail(LSW_E_ARG, "lsw_create: impl=%d invalid", c.impl);
  if (reinterpret_cast<uintptr_t>(router_w) % 16) return fail(LSW_E_ARG, "lsw_create: router_w not 16-byte aligned");
  for (int k = 0; k < LSW_NKIND; ++k) {
    const lsw_kind_desc& d = kinds[k];
    if (!d.W || !d.A || !d.B) return fail(LSW_E_ARG, "lsw_create: kind %s has a null pointer", kKindName[k]);
    if (d.d_out < 1 || d.d_in < 1) return fail(LSW_E_SHAPE, "lsw_create: kind %s shape %lldx%lld invalid", kKindName[k], (long long)d.d_out, (long long)d.d_in);
    if (d.d_in % 8) return fail(LSW_E_SHAPE, "lsw_create: kind %s d_in=%lld is not a multiple of 8", kKindName[k], (long long)d.d_in);
    if (d.d_in > 16384) return fail(LSW_E_SHAPE, "lsw_create: kind %s d_in=%lld > 16384", kKindName[k], (long long)d.d_in);
    if (reinterpret_cast<uintptr_t>(d.W) % 16 || reinterpret_cast<uintptr_t>(d.A) % 16 ||
        reinterpret_cast<uintptr_t>(d.B) % 16)
      return fail(LSW_E_ARG, "lsw_create: kind %s pointers must be 16-byte aligned", kKindName[k]);
  }
  // Group members share x: their d_in must agree.
  for (int g = 0; g < LSW_NGROUP; ++g)
    for (int i = 1; i < kGroupSize[g]; ++i)
      if (kinds[kGroupKinds[g][i]].d_in != kinds[kGroupKinds[g][0]].d_in)
        return fail(LSW_E_SHAPE, "lsw_create: kinds %s and %s share an input but d_in %lld != %lld",
                    kKindName[kGroupKinds[g][0]], kKindName[kGroupKinds[g][i]],
                    (long long)kinds[kGroupKinds[g][0]].d_in, (long long)kinds[kGroupKinds[g][i]].d_in);
  if (kinds[LSW_Q].d_in != c.d_model)
    return fail(LSW_E_SHAPE, "lsw_create: q d_in=%lld != d_model=%lld (x1 is the q/k/v input, R7)",
                (long long)kinds[LSW_Q].d_in, (long long)c.d_model);

  int impl = c.impl;
  if (impl == LSW_IMPL_AUTO) impl = c.dtype == LSW_BF16 ? LSW_IMPL_TC : LSW_IMPL_SIMT;
  if (impl == LSW_IMPL_TC && c.dtype != LSW_BF16)
    return fail(LSW_E_UNSUPPORTED, "lsw_create: the tensor-core switch needs bf16 storage");

  lsw_ctx* ctx = new lsw_ctx();
  ctx->cfg = c;
  memcpy(ctx->kinds, kinds, sizeof(ctx->kinds));
  ctx->router_w = router_w;
  ctx->impl = impl;
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "lsw_create: cudaGetDevice"); }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  ctx->gemv.grid_cap = ctx->num_sms;
  { const long x = opt_int("gemv_grid", 0); if (x >= 1 && x < ctx->gemv.grid_cap) ctx->gemv.grid_cap = (int)x; }
  { const long x = opt_int("gemv_op_kb", 0); if (x >= 4 && x <= 96) ctx->gemv.op_bytes = ctx->gemv.op_min = (uint32_t)x * 1024; }
  { const long x = opt_int("gemv_smem_kb", 0); if (x >= 32 && x <= 224) ctx->gemv.budget = ctx->gemv.budget_lora = (size_t)x * 1024; }
  { const char* v = opt_str("gemv"); ctx->gemv.ldg = v && strcmp(v, "ldg") == 0; }
  { const long v = opt_int("gemv_split", 1); ctx->gemv.split_rows = v < 0 || v > 2 ? 1 : (int)v; }
  ctx->gemv.probe = (int)probe_int("gemv_probe");
  ctx->host_graph = opt_int("host_graph", 1) != 0;
#ifdef LSW_TUNING
  { const char* v = opt_str("gemv_trace_buf"); if (v) gemv_set_trace(reinterpret_cast<uint32_t*>(strtoull(v, nullptr, 10))); }
#endif
  ctx->unmerged_flags = (int)probe_int("unmerged_flags");
  e = cudaMalloc(&ctx->d_state, sizeof(DevState));
  if (e != cudaSuccess) { delete ctx; return fail(LSW_E_OOM, "lsw_create: cudaMalloc(state) failed"); }
  e = cudaMemset(ctx->d_state, 0, sizeof(DevState));
  if (e != cudaSuccess) { lsw_destroy(ctx); return cuda_fail(e, "lsw_create: cudaMemset"); }
  fill_switch_params(ctx, ctx->simt_geom, kSimtTM, kSimtTN);
  if (impl == LSW_IMPL_TC) {
    const char* why = "";
    e = tc_plan_create(&ctx->tc, ctx->simt_geom, ctx->num_sms, &why);
    if (e != cudaSuccess || !ctx->tc) {
      lsw_destroy(ctx);
      if (e == cudaErrorMemoryAllocation) return fail(LSW_E_OOM, "lsw_create: packing LoRA operands: out of memory");
      if (e == cudaErrorNotSupported) return fail(LSW_E_UNSUPPORTED, "lsw_create: tensor-core switch: %s", why);
      return fail(LSW_E_CUDA, "lsw_create: tensor-core plan: %s (%s)", why, cudaGetErrorString(e));
    }
  }
  // token I/O layout
  int64_t xo = 0, yo = 0;
  for (int g = 0; g < LSW_NGROUP; ++g) {
    ctx->x_off[g] = xo;
    ctx->y_off[g] = yo;
    xo += kinds[kGroupKinds[g][0]].d_in;
    for (int i = 0; i < kGroupSize[g]; ++i) yo += kinds[kGroupKinds[g][i]].d_out;
  }
  ctx->x_per_layer = xo;
  ctx->y_per_layer = yo;
  ctx->xs_elems = xo * c.n_layers;
  ctx->ys_elems = yo * c.n_layers;
  *out = ctx;
  return LSW_OK;
}

lsw_status lsw_destroy(lsw_ctx* ctx) {
  if (!ctx) return fail(LSW_E_ARG, "lsw_destroy: null ctx");
  cudaDeviceSynchronize();
  if (ctx->comm) nccl()->CommDestroy(ctx->comm);
  if (ctx->tc) tc_plan_destroy(ctx->tc);
  cudaFree(ctx->lora_u);
  cudaFree(ctx->d_state);
  cudaFree(ctx->st_x1);
  cudaFree(ctx->st_xs);
  cudaFree(ctx->st_ys);
  cudaFree(ctx->st_idx);
  cudaFree(ctx->st_gate);
  for (cudaEvent_t ev : ctx->st_ev) cudaEventDestroy(ev);
  for (auto& hg : ctx->hgraph) if (hg.exec) cudaGraphExecDestroy(hg.exec);
  if (ctx->st_cap) cudaStreamDestroy(ctx->st_cap);
  pf_plan_destroy(ctx->pf);
  cudaFree(ctx->prefill_u);
  cudaFree(ctx->prefill_z);
  if (ctx->st_side) cudaStreamDestroy(ctx->st_side);
  delete ctx;
  return LSW_OK;
}

lsw_status lsw_get_info(const lsw_ctx* ctx, lsw_info* info) {
  if (!ctx || !info) return fail(LSW_E_ARG, "lsw_get_info: null argument");
  memset(info, 0, sizeof(*info));
  info->switch_impl = ctx->impl;
  if (ctx->impl == LSW_IMPL_TC) {
    info->tiles_total = tc_plan_tiles(ctx->tc);
    info->grid = tc_plan_grid(ctx->tc);
    info->tile_m = 128;
    info->tile_n = tc_plan_tile_n(ctx->tc);
    info->packed_bytes = tc_plan_bytes(ctx->tc);
    info->switch_kernel = tc_plan_kernel(ctx->tc);
  } else {
    info->tiles_total = ctx->simt_geom.tiles_total;
    info->grid = ctx->num_sms * 4;
    info->tile_m = kSimtTM;
    info->tile_n = kSimtTN;
  }
  info->merged = ctx->merged;
  info->num_sms = ctx->num_sms;
  info->kernel_launches = ctx->launches;
  info->xs_elems = ctx->xs_elems;
  info->ys_elems = ctx->ys_elems;
  return LSW_OK;
}

lsw_status lsw_nccl_version(int32_t* version, char* path, int64_t path_len) {
  if (!version) return fail(LSW_E_ARG, "lsw_nccl_version: null version");
  const Nccl* n = nccl();
  if (!n) return fail(LSW_E_NCCL, "lsw_nccl_version: libnccl.so.2 could not be loaded (%s)", dlerror());
  int v = 0;
  ncclResult_t r = n->GetVersion(&v);
  if (r != ncclSuccess) return fail(LSW_E_NCCL, "ncclGetVersion: %s", n->GetErrorString(r));
  *version = v;
  if (path && path_len > 0) {
    strncpy(path, n->path.c_str(), (size_t)path_len - 1);
    path[path_len - 1] = 0;
  }
  return LSW_OK;
}

lsw_status lsw_nccl_get_unique_id(void* id_out) {
  if (!id_out) return fail(LSW_E_ARG, "lsw_nccl_get_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  const Nccl* n = nccl();
  if (!n) return fail(LSW_E_NCCL, "lsw_nccl_get_unique_id: libnccl.so.2 could not be loaded");
  ncclResult_t r = n->GetUniqueId(reinterpret_cast<ncclUniqueId*>(id_out));
  if (r != ncclSuccess) return fail(LSW_E_NCCL, "ncclGetUniqueId: %s", n->GetErrorString(r));
  return LSW_OK;
}

lsw_status lsw_attach_nccl(lsw_ctx* ctx, const void* id) {
  if (!ctx || !id) return fail(LSW_E_ARG, "lsw_attach_nccl: null argument");
  if (ctx->comm) return fail(LSW_E_STATE, "lsw_attach_nccl: communicator already attached");
  const Nccl* n = nccl();
  if (!n) return fail(LSW_E_NCCL, "lsw_attach_nccl: libnccl.so.2 could not be loaded");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = n->CommInitRank(&ctx->comm, ctx->cfg.tp_size, uid, ctx->cfg.tp_rank);
  if (r != ncclSuccess) { ctx->comm = nullptr; return fail(LSW_E_NCCL, "ncclCommInitRank: %s", n->GetErrorString(r)); }
  return LSW_OK;
}

lsw_status lsw_router_topk(lsw_ctx* ctx, const void* x1, int32_t* idx, float* gate, void* stream) {
  if (!ctx || !x1 || !idx || !gate) return fail(LSW_E_ARG, "lsw_router_topk: null argument");
  cudaError_t e = launch_router(ctx->router_w, x1, ctx->cfg.n_experts, ctx->cfg.d_model, ctx->cfg.top_k,
                                ctx->cfg.dtype, idx, gate, ctx->d_state, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_router_topk: launch");
  ++ctx->launches;
  return LSW_OK;
}

static lsw_status run_switch(lsw_ctx* ctx, int mode, const int32_t* idx, const float* gate, cudaStream_t s) {
  SwitchParams p = ctx->simt_geom;
  p.mode = mode;
  p.cur_idx = idx;
  p.cur_g = gate;
  p.state = ctx->d_state;
  cudaError_t e;
  if (ctx->impl == LSW_IMPL_TC)
    e = launch_switch_tc(ctx->tc, p, s);
  else
    e = launch_switch_simt(p, ctx->cfg.dtype, ctx->num_sms * 4, s);
  if (e != cudaSuccess) return cuda_fail(e, "switch kernel launch");
  ++ctx->launches;
  return LSW_OK;
}

lsw_status lsw_merge_all_layers(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream) {
  if (!ctx || !idx || !gate) return fail(LSW_E_ARG, "lsw_merge_all_layers: null argument");
  lsw_status st = run_switch(ctx, ctx->merged ? MODE_SWITCH : MODE_MERGE, idx, gate, (cudaStream_t)stream);
  if (st == LSW_OK) ctx->merged = true;
  return st;
}

lsw_status lsw_attach_pristine(lsw_ctx* ctx, const void* const P[LSW_NKIND]) {
  if (!ctx || !P) return fail(LSW_E_ARG, "lsw_attach_pristine: null argument");
  for (int k = 0; k < LSW_NKIND; ++k) {
    if (!P[k]) return fail(LSW_E_ARG, "lsw_attach_pristine: kind %s: null pointer", kKindName[k]);
    if (reinterpret_cast<uintptr_t>(P[k]) % 16)
      return fail(LSW_E_ARG, "lsw_attach_pristine: kind %s: pointer not 16-byte aligned", kKindName[k]);
  }
  for (int k = 0; k < LSW_NKIND; ++k) ctx->simt_geom.kind[k].P = P[k];
  if (ctx->tc) {
    cudaError_t e = tc_plan_set_pristine(ctx->tc, ctx->simt_geom);
    if (e != cudaSuccess) {
      for (int k = 0; k < LSW_NKIND; ++k) ctx->simt_geom.kind[k].P = nullptr;
      return fail(LSW_E_ARG, "lsw_attach_pristine: cuTensorMapEncodeTiled failed");
    }
  }
  ctx->has_pristine = true;
  return LSW_OK;
}

lsw_status lsw_restore_merge_all_layers(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream) {
  if (!ctx || !idx || !gate) return fail(LSW_E_ARG, "lsw_restore_merge_all_layers: null argument");
  if (!ctx->has_pristine) return fail(LSW_E_STATE, "lsw_restore_merge_all_layers: no pristine copy attached");
  lsw_status st = run_switch(ctx, MODE_RESTORE, idx, gate, (cudaStream_t)stream);
  if (st == LSW_OK) ctx->merged = true;
  return st;
}

lsw_status lsw_unmerge_all_layers(lsw_ctx* ctx, void* stream) {
  if (!ctx) return fail(LSW_E_ARG, "lsw_unmerge_all_layers: null ctx");
  if (!ctx->merged) return fail(LSW_E_STATE, "lsw_unmerge_all_layers: nothing is merged");
  lsw_status st = run_switch(ctx, MODE_UNMERGE, nullptr, nullptr, (cudaStream_t)stream);
  if (st == LSW_OK) ctx->merged = false;
  return st;
}

static lsw_status gemv_sites(lsw_ctx* ctx, int layer, const int* kinds, int n, const void* x, float* y,
                             cudaStream_t s, const char* who, bool early_w = false) {
  if (!ctx || !x || !y) return fail(LSW_E_ARG, "%s: null argument", who);
  if (layer < 0 || layer >= ctx->cfg.n_layers)
    return fail(LSW_E_ARG, "%s: layer=%d not in [0,%d)", who, layer, ctx->cfg.n_layers);
  if (reinterpret_cast<uintptr_t>(x) % 16) return fail(LSW_E_ARG, "%s: x not 16-byte aligned", who);
  GemvParams p{};
  int64_t rows = 0;
  for (int i = 0; i < n; ++i) {
    const lsw_kind_desc& d = ctx->kinds[kinds[i]];
    p.site[i].W = (const uint8_t*)d.W + (size_t)layer * d.d_out * d.d_in * esize(ctx);
    p.site[i].d_out = d.d_out;
    p.site[i].row_begin = rows;
    rows += d.d_out;
  }
  p.n_sites = n;
  p.rows_total = rows;
  p.d_in = ctx->kinds[kinds[0]].d_in;
  p.x = x;
  p.y = y;
  // Row-parallel kinds under TP need the communicator: checked before anything
  // is enqueued (header contract).  A tp_size = 1 ctx with a (1-rank)
  // communicator attached all-reduces too: the identity, through the same call.
  const bool row_par = ctx->kinds[kinds[0]].row_parallel != 0;
  if (row_par && ctx->cfg.tp_size > 1 && !ctx->comm)
    return fail(LSW_E_NCCL, "%s: tp_size=%d but no NCCL communicator attached", who, ctx->cfg.tp_size);
  const bool allreduce = row_par && ctx->comm;
  cudaError_t e = launch_gemv(p, ctx->cfg.dtype, ctx->gemv, s, early_w);
  if (e != cudaSuccess) return cuda_fail(e, "decode GEMV launch");
  ++ctx->launches;
  // Row-parallel kinds under TP: partial sums -> allreduce.
  if (allreduce) {
    const Nccl* nc = nccl();
    ncclResult_t r = nc->AllReduce(y, y, (size_t)rows, ncclFloat, ncclSum, ctx->comm, s);
    if (r != ncclSuccess) return fail(LSW_E_NCCL, "%s: ncclAllReduce: %s", who, nc->GetErrorString(r));
  }
  return LSW_OK;
}

static lsw_status gemv_unmerged(lsw_ctx* ctx, int layer, int group, const void* x, float* y, const int32_t* idx,
                                const float* gate, cudaStream_t s, const char* who, bool early_w) {
  if (!ctx || !x || !y || !idx || !gate) return fail(LSW_E_ARG, "%s: null argument", who);
  if (layer < 0 || layer >= ctx->cfg.n_layers)
    return fail(LSW_E_ARG, "%s: layer=%d not in [0,%d)", who, layer, ctx->cfg.n_layers);
  if (group < 0 || group >= LSW_NGROUP) return fail(LSW_E_ARG, "%s: group=%d invalid", who, group);
  if (reinterpret_cast<uintptr_t>(x) % 16) return fail(LSW_E_ARG, "%s: x not 16-byte aligned", who);
  if (ctx->merged) return fail(LSW_E_STATE, "%s: the ctx is merged (unmerged decode reads the pristine W)", who);
  // Tensor parallelism: a column-parallel group's rows are complete on each
  // rank (x and A whole, W / B rows of the shard); a row-parallel kind (o,
  // down) holds W[:, shard] and A[:, shard], and its partial
  // W_s x_s + sum_j c_j B_j (A_j,s x_s) sums over the ranks to W x + sum_j c_j
  // B_j (A_j x) -- Eq. 2 is linear in the shards -- so the same all-reduce as
  // the merged decode's finishes it.  Checked before anything is enqueued.
  const bool row_par = ctx->kinds[kGroupKinds[group][0]].row_parallel != 0;
  if (row_par && ctx->cfg.tp_size > 1 && !ctx->comm)
    return fail(LSW_E_NCCL, "%s: tp_size=%d but no NCCL communicator attached", who, ctx->cfg.tp_size);
  if (!ctx->lora_u) {
    const size_t n = (size_t)3 * ctx->cfg.top_k * ctx->cfg.rank;
    if (cudaMalloc(&ctx->lora_u, n * sizeof(float)) != cudaSuccess)
      return fail(LSW_E_OOM, "%s: scratch allocation failed", who);
  }
  const size_t es = esize(ctx);
  GemvParams p{};
  GemvLora L{};
  int64_t rows = 0;
  const int n = kGroupSize[group];
  for (int i = 0; i < n; ++i) {
    const lsw_kind_desc& d = ctx->kinds[kGroupKinds[group][i]];
    p.site[i].W = (const uint8_t*)d.W + (size_t)layer * d.d_out * d.d_in * es;
    p.site[i].d_out = d.d_out;
    p.site[i].row_begin = rows;
    rows += d.d_out;
    L.A[i] = (const uint8_t*)d.A + (size_t)layer * ctx->cfg.n_experts * ctx->cfg.rank * d.d_in * es;
    L.B[i] = (const uint8_t*)d.B + (size_t)layer * ctx->cfg.n_experts * d.d_out * ctx->cfg.rank * es;
  }
  p.n_sites = n;
  p.rows_total = rows;
  p.d_in = ctx->kinds[kGroupKinds[group][0]].d_in;
  p.x = x;
  p.y = y;
  L.idx = idx;
  L.gate = gate;
  L.scale = ctx->cfg.alpha / (float)ctx->cfg.rank;
  L.k = ctx->cfg.top_k;
  L.r = ctx->cfg.rank;
  L.n_experts = ctx->cfg.n_experts;
  L.err = &ctx->d_state->err;
  L.u = ctx->lora_u;
  L.arrive = &ctx->d_state->lora_arrive;
  L.depart = &ctx->d_state->lora_depart;
  L.flags = ctx->unmerged_flags;
  cudaError_t e = launch_gemv(p, ctx->cfg.dtype, ctx->gemv, s, early_w, &L);
  if (e == cudaErrorNotSupported) return fail(LSW_E_UNSUPPORTED, "%s: needs the bulk GEMV (option gemv=ldg set)", who);
  if (e != cudaSuccess) return cuda_fail(e, "unmerged decode GEMV launch");
  ctx->launches += 1;                       // LoRA-down, GEMV and LoRA-up in one launch
  if (row_par && ctx->comm) {
    const Nccl* nc = nccl();
    ncclResult_t r = nc->AllReduce(y, y, (size_t)rows, ncclFloat, ncclSum, ctx->comm, s);
    if (r != ncclSuccess) return fail(LSW_E_NCCL, "%s: ncclAllReduce: %s", who, nc->GetErrorString(r));
  }
  return LSW_OK;
}

lsw_status lsw_decode_group_unmerged(lsw_ctx* ctx, int32_t layer, int32_t group, const void* x, float* y,
                                     const int32_t* idx, const float* gate, void* stream) {
  return gemv_unmerged(ctx, layer, group, x, y, idx, gate, (cudaStream_t)stream, "lsw_decode_group_unmerged",
                       /*early_w=*/true);
}

lsw_status lsw_prefill_group(lsw_ctx* ctx, int32_t layer, int32_t group, const void* X, int64_t T,
                             const int32_t* idx, const float* gate, float* Y, void* stream) {
  const char* who = "lsw_prefill_group";
  if (!ctx || !X || !idx || !gate || !Y) return fail(LSW_E_ARG, "%s: null argument", who);
  if (T < 1 || T > (1 << 20)) return fail(LSW_E_ARG, "%s: T=%lld not in [1, 2^20]", who, (long long)T);
  if (layer < 0 || layer >= ctx->cfg.n_layers)
    return fail(LSW_E_ARG, "%s: layer=%d not in [0,%d)", who, layer, ctx->cfg.n_layers);
  if (group < 0 || group >= LSW_NGROUP) return fail(LSW_E_ARG, "%s: group=%d invalid", who, group);
  if (ctx->merged) return fail(LSW_E_STATE, "%s: the ctx is merged (prefill reads the pristine W)", who);
  // tensor parallelism: as the unmerged decode -- column-parallel rows are
  // complete per rank, row-parallel partial outputs all-reduced (Eq. 2 is
  // linear in the d_in shards of W and A)
  const bool row_par = ctx->kinds[kGroupKinds[group][0]].row_parallel != 0;
  if (row_par && ctx->cfg.tp_size > 1 && !ctx->comm)
    return fail(LSW_E_NCCL, "%s: tp_size=%d but no NCCL communicator attached", who, ctx->cfg.tp_size);
  if (reinterpret_cast<uintptr_t>(X) % 16) return fail(LSW_E_ARG, "%s: X not 16-byte aligned", who);
  const bool tc = ctx->tc != nullptr;
  if (tc && !ctx->pf) {
    cudaError_t e = pf_plan_create(&ctx->pf, ctx->simt_geom, ctx->tc, ctx->num_sms);
    if (e != cudaSuccess) return cuda_fail(e, "lsw_prefill_group: tensor-core prefill plan");
  }
  const int n = kGroupSize[group];
  int64_t need_u = T * n * ctx->cfg.top_k * ctx->cfg.rank, need_z = 0;
  if (tc) pf_scratch(ctx->pf, n, T, &need_u, &need_z);
  if (need_u > ctx->prefill_u_elems) {
    cudaFree(ctx->prefill_u);
    ctx->prefill_u = nullptr;
    ctx->prefill_u_elems = 0;
    if (cudaMalloc(&ctx->prefill_u, need_u * sizeof(float)) != cudaSuccess)
      return fail(LSW_E_OOM, "%s: scratch allocation failed", who);
    ctx->prefill_u_elems = need_u;
  }
  if (need_z > ctx->prefill_z_elems) {
    cudaFree(ctx->prefill_z);
    ctx->prefill_z = nullptr;
    ctx->prefill_z_elems = 0;
    if (cudaMalloc(&ctx->prefill_z, need_z * 2) != cudaSuccess)
      return fail(LSW_E_OOM, "%s: scratch allocation failed", who);
    // the fused LoRA-down writes only the slots rho < r; the padding slots
    // (rho in [r, rp)) meet zero B columns and must hold finite values
    if (cudaMemset(ctx->prefill_z, 0, need_z * 2) != cudaSuccess)
      return fail(LSW_E_CUDA, "%s: scratch initialisation failed", who);
    ctx->prefill_z_elems = need_z;
  }
  const size_t es = esize(ctx);
  PrefillParams P{};
  int64_t rows = 0;
  int kinds[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const int kd = kGroupKinds[group][i];
    const lsw_kind_desc& d = ctx->kinds[kd];
    kinds[i] = kd;
    P.W[i] = (const uint8_t*)d.W + (size_t)layer * d.d_out * d.d_in * es;
    P.A[i] = (const uint8_t*)d.A + (size_t)layer * ctx->cfg.n_experts * ctx->cfg.rank * d.d_in * es;
    P.B[i] = (const uint8_t*)d.B + (size_t)layer * ctx->cfg.n_experts * d.d_out * ctx->cfg.rank * es;
    P.d_out[i] = d.d_out;
    P.row_begin[i] = rows;
    rows += d.d_out;
  }
  P.n_sites = n;
  P.k = ctx->cfg.top_k;
  P.r = ctx->cfg.rank;
  P.n_experts = ctx->cfg.n_experts;
  P.d_in = ctx->kinds[kGroupKinds[group][0]].d_in;
  P.rows = rows;
  P.T = T;
  P.scale = ctx->cfg.alpha / (float)ctx->cfg.rank;
  P.X = X;
  P.idx = idx;
  P.gate = gate;
  P.U = ctx->prefill_u;
  P.u_elems = ctx->prefill_u_elems;
  P.Z = ctx->prefill_z;
  P.Y = Y;
  cudaError_t e = tc ? launch_prefill_tc(ctx->pf, P, layer, kinds, (cudaStream_t)stream)
                     : launch_prefill_simt(P, ctx->cfg.dtype, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_prefill_group: launch");
  ctx->launches += tc ? 3 : 2;              // tc: LoRA-down GEMM, Z build, dense + LoRA-up GEMM
  if (row_par && ctx->comm) {
    const Nccl* nc = nccl();
    ncclResult_t r = nc->AllReduce(Y, Y, (size_t)(T * rows), ncclFloat, ncclSum, ctx->comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return fail(LSW_E_NCCL, "%s: ncclAllReduce: %s", who, nc->GetErrorString(r));
  }
  return LSW_OK;
}

lsw_status lsw_decode_all_layers_unmerged(lsw_ctx* ctx, const void* xs, float* ys, const int32_t* idx,
                                          const float* gate, void* stream) {
  if (!ctx || !xs || !ys || !idx || !gate) return fail(LSW_E_ARG, "lsw_decode_all_layers_unmerged: null argument");
  if (ctx->merged) return fail(LSW_E_STATE, "lsw_decode_all_layers_unmerged: the ctx is merged");
  const size_t es = esize(ctx);
  for (int l = 0; l < ctx->cfg.n_layers; ++l)
    for (int g = 0; g < LSW_NGROUP; ++g) {
      const uint8_t* xp = (const uint8_t*)xs + (size_t)(l * ctx->x_per_layer + ctx->x_off[g]) * es;
      float* yp = ys + l * ctx->y_per_layer + ctx->y_off[g];
      // W is never written on this path: every launch may prefetch it under PDL
      lsw_status st = gemv_unmerged(ctx, l, g, xp, yp, idx, gate, (cudaStream_t)stream,
                                    "lsw_decode_all_layers_unmerged", /*early_w=*/true);
      if (st != LSW_OK) return st;
    }
  return LSW_OK;
}

lsw_status lsw_decode_linear(lsw_ctx* ctx, int32_t layer, int32_t kind, const void* x, float* y, void* stream) {
  if (!ctx) return fail(LSW_E_ARG, "lsw_decode_linear: null ctx");
  if (kind < 0 || kind >= LSW_NKIND) return fail(LSW_E_ARG, "lsw_decode_linear: kind=%d invalid", kind);
  int k = kind;
  return gemv_sites(ctx, layer, &k, 1, x, y, (cudaStream_t)stream, "lsw_decode_linear");
}

lsw_status lsw_decode_group(lsw_ctx* ctx, int32_t layer, int32_t group, const void* x, float* y, void* stream) {
  if (!ctx) return fail(LSW_E_ARG, "lsw_decode_group: null ctx");
  if (group < 0 || group >= LSW_NGROUP) return fail(LSW_E_ARG, "lsw_decode_group: group=%d invalid", group);
  return gemv_sites(ctx, layer, kGroupKinds[group], kGroupSize[group], x, y, (cudaStream_t)stream,
                    "lsw_decode_group");
}

lsw_status lsw_decode_token(lsw_ctx* ctx, const void* x1, const void* xs, float* ys, int32_t* idx, float* gate,
                            void* stream) {
  if (!ctx || !x1 || !xs || !ys || !idx || !gate) return fail(LSW_E_ARG, "lsw_decode_token: null argument");
  lsw_status st = lsw_router_topk(ctx, x1, idx, gate, stream);                       // Alg. 1 l.1
  if (st != LSW_OK) return st;
  st = lsw_merge_all_layers(ctx, idx, gate, stream);                                   // l.2-4
  if (st != LSW_OK) return st;
  return lsw_decode_all_layers(ctx, xs, ys, stream);                                  // l.5
}

lsw_status lsw_decode_all_layers(lsw_ctx* ctx, const void* xs, float* ys, void* stream) {
  if (!ctx || !xs || !ys) return fail(LSW_E_ARG, "lsw_decode_all_layers: null argument");
  if (reinterpret_cast<uintptr_t>(xs) % 16) return fail(LSW_E_ARG, "lsw_decode_all_layers: xs not 16-byte aligned");
  const size_t es = esize(ctx);
  for (int l = 0; l < ctx->cfg.n_layers; ++l)
    for (int g = 0; g < LSW_NGROUP; ++g) {
      const uint8_t* xp = (const uint8_t*)xs + (size_t)(l * ctx->x_per_layer + ctx->x_off[g]) * es;
      float* yp = ys + l * ctx->y_per_layer + ctx->y_off[g];
      // every GEMV but the first may prefetch W under PDL (the first may follow the switch)
      lsw_status st = gemv_sites(ctx, l, kGroupKinds[g], kGroupSize[g], xp, yp, (cudaStream_t)stream,
                                 "lsw_decode_all_layers", /*early_w=*/l > 0 || g > 0);
      if (st != LSW_OK) return st;
    }
  return LSW_OK;
}

lsw_status lsw_decode_token_fused(lsw_ctx* ctx, const void* x1, const void* xs, float* ys, int32_t* idx,
                                  float* gate, void* stream) {
  if (!ctx || !x1 || !xs || !ys || !idx || !gate) return fail(LSW_E_ARG, "lsw_decode_token_fused: null argument");
  if (reinterpret_cast<uintptr_t>(xs) % 16) return fail(LSW_E_ARG, "lsw_decode_token_fused: xs not 16-byte aligned");
  if (!ctx->tc || ctx->cfg.tp_size != 1)
    return fail(LSW_E_UNSUPPORTED, "lsw_decode_token_fused: needs the tensor-core switch and tp_size == 1");
  if (!ctx->fused_ready) {
    int nk[LSW_NGROUP];
    for (int g = 0; g < LSW_NGROUP; ++g) nk[g] = kGroupSize[g];
    cudaError_t e = tc_plan_set_fused(ctx->tc, ctx->cfg.n_layers, ctx->x_off, ctx->y_off, ctx->x_per_layer,
                                      ctx->y_per_layer, kGroupKinds, nk);
    if (e == cudaErrorNotSupported)
      return fail(LSW_E_UNSUPPORTED, "lsw_decode_token_fused: the fused decode is built on the shared-memory fold (switch_kernel 3), and this ctx switches with another mode (per-term for its rank / top-k, or the TMEM strip option)");
    if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_fused: segment table");
    ctx->fused_ready = true;
  }
  cudaStream_t s = (cudaStream_t)stream;
  lsw_status st = lsw_router_topk(ctx, x1, idx, gate, stream);                       // Alg. 1 l.1
  if (st != LSW_OK) return st;
  cudaError_t e = cudaMemsetAsync(ys, 0, ctx->ys_elems * sizeof(float), s);         // accumulated
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_fused: memset");
  SwitchParams p = ctx->simt_geom;
  p.mode = ctx->merged ? MODE_SWITCH : MODE_MERGE;                                   // l.2-5, one launch
  p.cur_idx = idx;
  p.cur_g = gate;
  p.state = ctx->d_state;
  e = launch_switch_tc_fused(ctx->tc, p, s, xs, ys);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_fused: launch");
  ++ctx->launches;
  ctx->merged = true;
  return LSW_OK;
}

// The token's work from host buffers, enqueued on `s` (its side stream forked
// and joined back through events, so the whole sequence can be captured).
static lsw_status host_token_enqueue(lsw_ctx* ctx, const void* x1_h, const void* xs_h, float* ys_h, int32_t* idx_h,
                                     float* gate_h, cudaStream_t s) {
  const size_t es = esize(ctx);
  void* stream = (void*)s;
  cudaError_t e = cudaMemcpyAsync(ctx->st_x1, x1_h, ctx->cfg.d_model * es, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: H2D");
  cudaStream_t side = ctx->st_side;
  // the side stream starts after everything already on `s` (the previous
  // token's readers of st_xs / st_ys are done)
  e = cudaEventRecord(ctx->st_ev[0], s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ctx->st_ev[0], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->st_xs, xs_h, ctx->xs_elems * es, cudaMemcpyHostToDevice, side);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->st_ev[0], side);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: H2D");
  lsw_status st = lsw_router_topk(ctx, ctx->st_x1, ctx->st_idx, ctx->st_gate, stream);          // Alg. 1 l.1
  if (st != LSW_OK) return st;
  st = lsw_merge_all_layers(ctx, ctx->st_idx, ctx->st_gate, stream);                          // l.2-4
  if (st != LSW_OK) return st;
  e = cudaStreamWaitEvent(s, ctx->st_ev[0], 0);                                                 // xs landed
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: wait");
  for (int l = 0; l < ctx->cfg.n_layers; ++l) {                                                // l.5
    for (int g = 0; g < LSW_NGROUP; ++g) {
      const uint8_t* xp = (const uint8_t*)ctx->st_xs + (size_t)(l * ctx->x_per_layer + ctx->x_off[g]) * es;
      float* yp = ctx->st_ys + l * ctx->y_per_layer + ctx->y_off[g];
      st = gemv_sites(ctx, l, kGroupKinds[g], kGroupSize[g], xp, yp, s, "lsw_decode_token_host",
                      /*early_w=*/l > 0 || g > 0);
      if (st != LSW_OK) return st;
    }
    e = cudaEventRecord(ctx->st_ev[1 + l], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ctx->st_ev[1 + l], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ys_h + l * ctx->y_per_layer, ctx->st_ys + l * ctx->y_per_layer,
                          ctx->y_per_layer * sizeof(float), cudaMemcpyDeviceToHost, side);
    if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: D2H");
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(idx_h, ctx->st_idx, ctx->cfg.top_k * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(gate_h, ctx->st_gate, ctx->cfg.top_k * sizeof(float), cudaMemcpyDeviceToHost, s);
  // join the side stream back into `s`
  if (e == cudaSuccess) e = cudaEventRecord(ctx->st_ev[1 + ctx->cfg.n_layers], side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->st_ev[1 + ctx->cfg.n_layers], 0);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: D2H");
  return LSW_OK;
}

lsw_status lsw_decode_token_host(lsw_ctx* ctx, const void* x1_h, const void* xs_h, float* ys_h, int32_t* idx_h,
                                 float* gate_h, void* stream) {
  if (!ctx || !x1_h || !xs_h || !ys_h || !idx_h || !gate_h) return fail(LSW_E_ARG, "lsw_decode_token_host: null argument");
  const size_t es = esize(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  if (!ctx->st_x1) {
    if (cudaMalloc(&ctx->st_x1, ctx->cfg.d_model * es) != cudaSuccess ||
        cudaMalloc(&ctx->st_xs, ctx->xs_elems * es) != cudaSuccess ||
        cudaMalloc(&ctx->st_ys, ctx->ys_elems * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&ctx->st_idx, LSW_MAX_TOPK * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&ctx->st_gate, LSW_MAX_TOPK * sizeof(float)) != cudaSuccess)
      return fail(LSW_E_OOM, "lsw_decode_token_host: staging allocation failed");
  }
  // Copies overlap the token: x1 goes first on the token's stream (the router
  // needs it); the GEMV inputs on a side stream while the router and the
  // switch run; each layer's outputs go back on the side stream as soon as
  // that layer's GEMVs are done.
  if (!ctx->st_side) {
    if (cudaStreamCreateWithFlags(&ctx->st_side, cudaStreamNonBlocking) != cudaSuccess)
      return fail(LSW_E_CUDA, "lsw_decode_token_host: side stream");
    ctx->st_ev.resize(2 + ctx->cfg.n_layers);
    for (auto& ev : ctx->st_ev)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        return fail(LSW_E_CUDA, "lsw_decode_token_host: events");
  }
  // From the second call on, the token is ONE graph launch: its ~130 kernels
  // and copies enqueued once (captured on a ctx stream), so the host adds a
  // single launch per token.  One graph per state of the decision slot (the
  // first token merges, later ones switch); captured again if the host
  // buffers change.  The graph's kernels read the same device state (decision
  // slot, error latch) as the eager path.
  const int mode = ctx->merged ? 1 : 0;
  auto& hg = ctx->hgraph[mode];
  const void* key[5] = {x1_h, xs_h, ys_h, idx_h, gate_h};
  if (ctx->host_graph && ctx->host_calls > 0) {
    if (hg.exec && memcmp(hg.key, key, sizeof(key)) != 0) {
      cudaGraphExecDestroy(hg.exec);
      hg.exec = nullptr;
    }
    if (!hg.exec) {
      if (!ctx->st_cap && cudaStreamCreateWithFlags(&ctx->st_cap, cudaStreamNonBlocking) != cudaSuccess)
        return fail(LSW_E_CUDA, "lsw_decode_token_host: capture stream");
      const bool merged0 = ctx->merged;
      const uint64_t launches0 = ctx->launches;
      cudaError_t e = cudaStreamBeginCapture(ctx->st_cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: capture");
      lsw_status st = host_token_enqueue(ctx, x1_h, xs_h, ys_h, idx_h, gate_h, ctx->st_cap);
      cudaGraph_t graph = nullptr;
      e = cudaStreamEndCapture(ctx->st_cap, &graph);
      hg.launches = ctx->launches - launches0;
      ctx->merged = merged0;                       // nothing ran yet
      ctx->launches = launches0;
      if (st != LSW_OK) { if (graph) cudaGraphDestroy(graph); return st; }
      if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: capture");
      e = cudaGraphInstantiate(&hg.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) { hg.exec = nullptr; return cuda_fail(e, "lsw_decode_token_host: instantiate"); }
      memcpy(hg.key, key, sizeof(key));
    }
    cudaError_t e = cudaGraphLaunch(hg.exec, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: graph");
    ctx->merged = true;
    ctx->launches += hg.launches;
    ++ctx->host_calls;
    return LSW_OK;
  }
  lsw_status st = host_token_enqueue(ctx, x1_h, xs_h, ys_h, idx_h, gate_h, s);
  if (st != LSW_OK) return st;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_decode_token_host: D2H");
  ++ctx->host_calls;
  return LSW_OK;
}

lsw_status lsw_device_status(lsw_ctx* ctx, void* stream, int32_t* code) {
  if (!ctx) return fail(LSW_E_ARG, "lsw_device_status: null ctx");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_device_status: sync");
  int32_t err = 0;
  e = cudaMemcpy(&err, &ctx->d_state->err, sizeof(err), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "lsw_device_status: read latch");
  if (code) *code = err;
  if (err) {
    cudaMemset(&ctx->d_state->err, 0, sizeof(int32_t));
    return fail(LSW_E_DEVICE, "device error latched: code %d (%s)", err,
                err == LSW_DEV_NONFINITE_LOGITS ? "non-finite router logits"
                : err == LSW_DEV_BAD_INDEX      ? "expert index out of range or duplicated"
                                                : "non-finite gate");
  }
  return LSW_OK;
}

lsw_status lsw_debug_merge_per_matrix(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream) {
  if (!ctx || !idx || !gate) return fail(LSW_E_ARG, "lsw_debug_merge_per_matrix: null argument");
  if (ctx->merged) return fail(LSW_E_STATE, "lsw_debug_merge_per_matrix: the ctx is merged");
  if (!ctx->tc) return fail(LSW_E_UNSUPPORTED, "lsw_debug_merge_per_matrix: needs the tensor-core switch");
  SwitchParams p = ctx->simt_geom;
  p.mode = MODE_MERGE;
  p.cur_idx = idx;
  p.cur_g = gate;
  p.state = ctx->d_state;
  for (int k = 0; k < LSW_NKIND; ++k)
    for (int l = 0; l < ctx->cfg.n_layers; ++l) {
      int64_t t0 = 0;
      const int64_t n = tc_plan_matrix_tiles(ctx->tc, k, l, &t0);
      cudaError_t e = launch_switch_tc(ctx->tc, p, (cudaStream_t)stream, t0, n);
      if (e != cudaSuccess) return cuda_fail(e, "lsw_debug_merge_per_matrix: launch");
      ++ctx->launches;
    }
  ctx->merged = true;
  return LSW_OK;
}

lsw_status lsw_debug_set_option(const char* key, const char* value) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  if (!key) { g_opts.clear(); return LSW_OK; }
  if (!value) g_opts.erase(key);
  else g_opts[key] = value;
  return LSW_OK;
}

}  // extern "C"
