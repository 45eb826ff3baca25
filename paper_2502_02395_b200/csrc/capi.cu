// C ABI plumbing: error reporting, the native step executor and CUDA-graph
// capture of a whole factorization program (see include/h2ulv_b200.h).
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

static thread_local char g_err[512] = "";

int h2g_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int h2g_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return H2G_OK;
}

extern "C" const char* h2g_last_error(void) { return g_err; }
extern "C" int h2g_abi_version(void) { return H2G_ABI_VERSION; }

extern "C" int h2g_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

static int run_step(const h2g_step& s, cudaStream_t st) {
  switch (s.kind) {
    case H2G_STEP_GEMM_NN:
    case H2G_STEP_GEMM_NT:
    case H2G_STEP_GEMM_TN:
    case H2G_STEP_GEMM_TT: {
      int k = s.kind - H2G_STEP_GEMM_NN;
      if (s.npd)   /* deterministic split-K: arg = tile_cfg | nsplit << 8, npd = the workspace */
        return h2g_gemm_grouped_split(k >> 1, k & 1, s.arg & 0xff, (const h2g_gemm_problem*)s.descs, s.map, s.grid,
                                      s.arg >> 8, (void*)s.npd, st);
      if (s.aux)   /* per-problem extension (separate Cin / compact-WY relabel) */
        return h2g_gemm_grouped_ext(k >> 1, k & 1, s.arg, (const h2g_gemm_problem*)s.descs,
                                    (const h2g_gemm_ext*)s.aux, s.map, s.grid, st);
      return h2g_gemm_grouped(k >> 1, k & 1, s.arg, (const h2g_gemm_problem*)s.descs, s.map, s.grid, st);
    }
    case H2G_STEP_COPY:
      return h2g_block_copy((const h2g_copy_desc*)s.descs, s.map, s.grid, st);
    case H2G_STEP_MEMCPY: {
      if (s.count <= 0) return H2G_OK;
      cudaError_t e = cudaMemcpyAsync((void*)s.descs, (const void*)s.map, (size_t)s.count, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "memcpy step: %s", cudaGetErrorString(e));
      return H2G_OK;
    }
    case H2G_STEP_QR_PANEL:
      return h2g_qr_panel((const h2g_qr_panel_desc*)s.descs, s.count, s.arg, st);
    case H2G_STEP_BASIS:
      return h2g_basis_finish((const h2g_basis_desc*)s.descs, s.count, st);
    case H2G_STEP_GEMV:
      return h2g_gemv_grouped((const h2g_gemv_out*)s.descs, s.count, (const h2g_gemv_term*)s.map,
                              (const int32_t*)s.aux, s.grid, s.arg, st);
    case H2G_STEP_TRSV:
      return h2g_trsv_batched((const h2g_trsv_desc*)s.descs, s.count, s.arg, s.grid, st);  // grid = w
    case H2G_STEP_KBLOCK:
      return h2g_kernel_blocks((const h2g_kblock_desc*)s.descs, s.map, s.grid, (const double*)s.aux, s.arg,
                               s.d0, s.d1, (int64_t*)s.npd, st);
    case H2G_STEP_CHOL_PANEL:
      return h2g_chol_panel_sync((const h2g_chol_panel_desc*)s.descs, s.count, s.map, s.grid, s.npd,
                                 (int32_t*)s.aux, st);
    case H2G_STEP_TRSM_ROWS:
      return h2g_trsm_rows((const h2g_rows_desc*)s.descs, s.map, s.grid, st);
    case H2G_STEP_SYMCHECK:
      return h2g_sym_check((const h2g_symcheck_desc*)s.descs, s.count, (unsigned long long*)s.aux, st);
    case H2G_STEP_TRIINV:
      return h2g_tri_inv((const h2g_triinv_desc*)s.descs, s.map, s.grid, s.npd, st);
    case H2G_STEP_CHOL_BOX:
      return h2g_chol_box((const h2g_cholbox_desc*)s.descs, s.count, s.npd, st);
    case H2G_STEP_XFORM_T:
      return h2g_xform_t((const h2g_xform_desc*)s.descs, s.map, s.grid, s.arg, s.count < 0, st);
    case H2G_STEP_XFORM_N:
      return h2g_xform_n((const h2g_xform_n_desc*)s.descs, s.map, s.grid, s.arg, s.count < 0, (int)s.d0, st);
    case H2G_STEP_NOP:
      return H2G_OK;
    default:
      return h2g_set_error(H2G_ESTEP, "unknown step kind %d", s.kind);
  }
}

constexpr int kMaxLanes = 5;

// Lanes of a multi-lane program run on the context's own streams: lanes 0
// (the critical chain) and 1 (its look-ahead trailing updates) at the
// device's greatest stream priority, lanes 2..4 (work that only has to be
// done by the next merge / by the solve) at the least priority, so the block
// scheduler hands free SMs to the chain first and the side lanes fill the
// gaps of the latency-bound panel steps.  H2G_LANE_PRIORITY=0 gives every
// lane the default priority.  The caller's stream only forks and joins.
struct ExecCtx {
  cudaStream_t side[kMaxLanes] = {};
  std::vector<cudaEvent_t> ev;
  cudaEvent_t fork = nullptr, join[kMaxLanes] = {};
};

extern "C" int h2g_exec_ctx_create(int n_events, void** ctx_out) {
  if (!ctx_out || n_events < 0) return h2g_set_error(H2G_EINVAL, "h2g_exec_ctx_create: bad arguments");
  ExecCtx* c = new ExecCtx();
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const char* env = getenv("H2G_LANE_PRIORITY");
  if (env && env[0] == '0') least = greatest = 0;
  cudaError_t e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  for (int l = 0; l < kMaxLanes && e == cudaSuccess; ++l) {
    e = cudaStreamCreateWithPriority(&c->side[l], cudaStreamNonBlocking, l <= 1 ? greatest : least);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join[l], cudaEventDisableTiming);
  }
  c->ev.resize(n_events, nullptr);
  for (int i = 0; i < n_events && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    h2g_exec_ctx_destroy(c);
    return h2g_set_error(H2G_ECUDA, "h2g_exec_ctx_create: %s", cudaGetErrorString(e));
  }
  *ctx_out = c;
  return H2G_OK;
}

extern "C" int h2g_exec_ctx_destroy(void* ctx) {
  ExecCtx* c = (ExecCtx*)ctx;
  if (!c) return H2G_OK;
  for (cudaEvent_t e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->fork) cudaEventDestroy(c->fork);
  for (int l = 0; l < kMaxLanes; ++l) {
    if (c->join[l]) cudaEventDestroy(c->join[l]);
    if (c->side[l]) cudaStreamDestroy(c->side[l]);
  }
  delete c;
  return H2G_OK;
}

extern "C" int h2g_run_program(const h2g_step* steps, int nsteps, void* stream, void* ctx) {
  if (nsteps < 0 || (nsteps > 0 && !steps)) return h2g_set_error(H2G_EINVAL, "h2g_run_program: bad steps");
  cudaStream_t main_st = (cudaStream_t)stream;
  ExecCtx* c = (ExecCtx*)ctx;
  bool used[kMaxLanes] = {};
  bool multi = false;
  for (int i = 0; i < nsteps; ++i) {
    const int ln = steps[i].lane;
    if (ln < 0 || ln >= kMaxLanes) return h2g_set_error(H2G_EINVAL, "step %d: bad lane %d", i, ln);
    used[ln] = true;
    if (ln > 0 && c) multi = true;
  }
  if (multi) {  // fork: every lane starts after everything already queued on the caller's stream
    cudaEventRecord(c->fork, main_st);
    for (int l = 0; l < kMaxLanes; ++l)
      if (used[l]) cudaStreamWaitEvent(c->side[l], c->fork, 0);
  }
  for (int i = 0; i < nsteps; ++i) {
    const h2g_step& sp = steps[i];
    cudaStream_t st = multi ? c->side[sp.lane] : main_st;
    if (multi && sp.wait_ev >= 0) {
      if (sp.wait_ev >= (int)c->ev.size()) return h2g_set_error(H2G_EINVAL, "step %d: bad wait event", i);
      cudaStreamWaitEvent(st, c->ev[sp.wait_ev], 0);
    }
    int rc = run_step(sp, st);
    if (rc) {
      char buf[400];
      snprintf(buf, sizeof(buf), "%.380s", g_err);
      return h2g_set_error(rc, "step %d (kind %d): %s", i, sp.kind, buf);
    }
    if (multi && sp.rec_ev >= 0) {
      if (sp.rec_ev >= (int)c->ev.size()) return h2g_set_error(H2G_EINVAL, "step %d: bad record event", i);
      cudaEventRecord(c->ev[sp.rec_ev], st);
    }
  }
  if (multi) {  // join: the caller's stream continues only after every lane drained
    for (int l = 0; l < kMaxLanes; ++l)
      if (used[l]) {
        cudaEventRecord(c->join[l], c->side[l]);
        cudaStreamWaitEvent(main_st, c->join[l], 0);
      }
  }
  return H2G_OK;
}

extern "C" int h2g_run_program_timed(const h2g_step* steps, int nsteps, void* stream, float* out_ms) {
  if (nsteps <= 0) return H2G_OK;
  if (!steps || !out_ms) return h2g_set_error(H2G_EINVAL, "h2g_run_program_timed: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = new cudaEvent_t[nsteps + 1];
  for (int i = 0; i <= nsteps; ++i) cudaEventCreate(&ev[i]);
  int rc = H2G_OK;
  for (int i = 0; i < nsteps && rc == H2G_OK; ++i) {  // lanes ignored: serialized timing
    cudaEventRecord(ev[i], st);
    rc = run_step(steps[i], st);
  }
  cudaEventRecord(ev[nsteps], st);
  cudaEventSynchronize(ev[nsteps]);
  for (int i = 0; i < nsteps; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    out_ms[i] = ms;
  }
  for (int i = 0; i <= nsteps; ++i) cudaEventDestroy(ev[i]);
  delete[] ev;
  return rc;
}

extern "C" int h2g_graph_capture(const h2g_step* steps, int nsteps, void* stream, void* ctx, void** exec_out) {
  if (!exec_out) return h2g_set_error(H2G_EINVAL, "h2g_graph_capture: null exec_out");
  cudaStream_t st = (cudaStream_t)stream;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "begin capture: %s", cudaGetErrorString(e));
  int rc = h2g_run_program(steps, nsteps, stream, ctx);
  e = cudaStreamEndCapture(st, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "end capture: %s", cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "instantiate: %s", cudaGetErrorString(e));
  *exec_out = (void*)exec;
  return H2G_OK;
}

extern "C" int h2g_graph_launch(void* exec, void* stream) {
  if (!exec) return h2g_set_error(H2G_EINVAL, "h2g_graph_launch: null graph");
  cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream);
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "graph launch: %s", cudaGetErrorString(e));
  return H2G_OK;
}

extern "C" int h2g_graph_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return H2G_OK;
}

// ------------------------------------------------------------------ factorization session
struct Session {
  void* ctx = nullptr;
  cudaGraphExec_t graph = nullptr;
  int32_t* d_npd = nullptr;
  int depth = 0;
  std::vector<int32_t> slot_base;   // level l -> first slot (l = 0: the root)
  std::vector<int32_t> host;
};

extern "C" int h2g_session_create(const h2g_step* steps, int nsteps, int n_events, int32_t* d_npd, int depth,
                                  const int32_t* slot_base, void* stream, void** session_out) {
  if (!steps || nsteps <= 0 || !d_npd || !slot_base || depth < 0 || !session_out)
    return h2g_set_error(H2G_EINVAL, "h2g_session_create: bad arguments");
  Session* s = new Session();
  s->d_npd = d_npd;
  s->depth = depth;
  s->slot_base.assign(slot_base, slot_base + depth + 1);
  int rc = h2g_exec_ctx_create(n_events > 0 ? n_events : 1, &s->ctx);
  void* exec = nullptr;
  if (!rc) rc = h2g_graph_capture(steps, nsteps, stream, s->ctx, &exec);
  if (rc) {
    h2g_session_destroy(s);
    return rc;
  }
  s->graph = (cudaGraphExec_t)exec;
  int total = 0;
  for (int l = 0; l <= depth; ++l) total = std::max(total, slot_base[l] + (l ? (1 << l) : 1));
  s->host.resize(total);
  *session_out = s;
  return H2G_OK;
}

extern "C" int h2g_session_factor_async(void* session, void* stream) {
  Session* s = (Session*)session;
  if (!s || !s->graph) return h2g_set_error(H2G_EINVAL, "h2g_session_factor_async: null session");
  return h2g_graph_launch(s->graph, stream);
}

extern "C" int h2g_session_status(void* session, void* stream, h2g_npd_status* status) {
  Session* s = (Session*)session;
  if (!s || !status) return h2g_set_error(H2G_EINVAL, "h2g_session_status: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(s->host.data(), s->d_npd, s->host.size() * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return h2g_set_error(H2G_ECUDA, "h2g_session_status: %s", cudaGetErrorString(e));
  *status = h2g_npd_status{0, 0, 0, 0};
  for (int l = s->depth; l >= 0; --l) {          // deepest level first, then the root
    const int base = s->slot_base[l], cnt = l ? (1 << l) : 1;
    for (int b = 0; b < cnt; ++b)
      if (s->host[base + b] != INT32_MAX) {
        *status = h2g_npd_status{1, s->host[base + b], l, b};
        return h2g_set_error(H2G_ENPD, "non-positive pivot %d at level %d, box %d", s->host[base + b], l, b);
      }
  }
  return H2G_OK;
}

extern "C" int h2g_session_destroy(void* session) {
  Session* s = (Session*)session;
  if (!s) return H2G_OK;
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->ctx) h2g_exec_ctx_destroy(s->ctx);
  delete s;
  return H2G_OK;
}
