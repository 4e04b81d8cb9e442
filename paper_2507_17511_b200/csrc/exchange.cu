// Compressed exchanges as C-ABI objects (include/compactcomm.h, "exchange"):
// one patch-parallel / Ulysses layer step = K1 encode -> NCCL collective -> K2
// decode, stream-ordered, callable from C with no Python (the seam the
// reference's mesh.py:188-236 + transport.py:36-43 occupy).
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): inside a PyTorch process that
// resolves to the NCCL torch already loaded, so a communicator taken from
// ProcessGroupNCCL._comm_ptr() can be handed in; a C program gets its own through
// cc_comm_get_unique_id / cc_comm_init_rank.  The library itself does not link
// NCCL, so the encode/decode entry points load on machines without it.
//
// Layer objects own every device buffer of the step: the reconstruction
// (rows x cols f32; this rank's row shard is the sender base, mesh:233), the
// sender's feedback / ref, the codec workspace, the StepRecord and the send /
// receive wire buffers (registered with ncclCommRegister when available).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/compactcomm.h"
#include "cc_internal.h"
#include "nccl.h"

namespace cc {
namespace {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*CommRegister)(const ncclComm_t, void *, size_t, void **) = nullptr;
  ncclResult_t (*CommDeregister)(const ncclComm_t, void *) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

Nccl &nccl() {
  static Nccl api = [] {
    Nccl a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
      return a;
    }
    bool all = true;
    auto get = [&](auto &fn, const char *name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        a.why = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.CommCount, "ncclCommCount");
    get(a.CommUserRank, "ncclCommUserRank");
    get(a.AllGather, "ncclAllGather");
    get(a.Send, "ncclSend");
    get(a.Recv, "ncclRecv");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.GetErrorString, "ncclGetErrorString");
    // optional: buffer registration (user-buffer fast paths)
    a.CommRegister = reinterpret_cast<decltype(a.CommRegister)>(dlsym(h, "ncclCommRegister"));
    a.CommDeregister = reinterpret_cast<decltype(a.CommDeregister)>(dlsym(h, "ncclCommDeregister"));
    a.ok = all;
    return a;
  }();
  return api;
}

int nccl_status(ncclResult_t r, const char *where) {
  if (r == ncclSuccess) return CC_OK;
  set_error(std::string(where) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
  return CC_ERR_NCCL;
}

int need_nccl() {
  if (!nccl().ok) {
    set_error(nccl().why);
    return CC_ERR_NCCL;
  }
  return CC_OK;
}

bool quant(int codec) { return codec == CC_SIGN1 || codec == CC_QUANT2 || codec == CC_QUANT4; }

// exact body bytes of one compressed (non-warmup) transmission
int64_t body_of(const cc_codec_spec &s, int64_t rows, int64_t cols) {
  if (s.codec == CC_TOPK) return 6 * cc_topk_count(rows, cols, s.keep_fraction);
  if (s.codec == CC_NMBLOCK) return cc_body_bytes(CC_NMBLOCK, rows, cols, CC_NM_PARAM(s.nm_n, s.nm_m));
  return cc_body_bytes(s.codec, rows, cols, 0);
}

int64_t param_of(const cc_codec_spec &s, int64_t rows, int64_t cols) {
  if (s.codec == CC_TOPK) return cc_topk_count(rows, cols, s.keep_fraction);
  if (s.codec == CC_NMBLOCK) return CC_NM_PARAM(s.nm_n, s.nm_m);
  return 0;
}

int64_t ws_of(const cc_codec_spec &s, int64_t rows, int64_t cols) {
  if (s.codec == CC_RAW) return 0;
  return cc_workspace_bytes(s.codec, rows, cols, param_of(s, rows, cols));
}

int check_spec(const cc_codec_spec *s) {
  if (!s) {
    set_error("null codec spec");
    return CC_ERR_ARG;
  }
  if (!(quant(s->codec) || s->codec == CC_TOPK || s->codec == CC_NMBLOCK || s->codec == CC_RAW)) {
    set_error("exchange codecs: raw (identity), sign1, quant2, quant4, top-k, N:M");
    return CC_ERR_UNSUPPORTED;
  }
  if (s->scale_mode < CC_SCALE_RANK1 || s->scale_mode > CC_SCALE_PER_CHANNEL) {
    set_error("bad scale mode");
    return CC_ERR_ARG;
  }
  if (s->codec == CC_TOPK && !(s->keep_fraction > 0.0 && s->keep_fraction <= 1.0)) {
    set_error("top-k needs keep_fraction in (0, 1]");
    return CC_ERR_ARG;
  }
  if (s->codec == CC_NMBLOCK && !(1 <= s->nm_n && s->nm_n <= s->nm_m && s->nm_m <= 65535)) {
    set_error("N:M needs 1 <= n <= m <= 65535");
    return CC_ERR_ARG;
  }
  return CC_OK;
}

template <typename T>
int dalloc(T **p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) return CC_OK;
  if (cudaMalloc(reinterpret_cast<void **>(p), bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc failed");
    return CC_ERR_CUDA;
  }
  if (cudaMemset(*p, 0, bytes) != cudaSuccess) return cuda_status("cudaMemset");
  return CC_OK;
}

// receiver accumulate mode: replace for naive, "dense base + 0.0 then sparse add"
// for the first top-k add after a replace (the reference's dense add, pl:163)
int receiver_acc(const cc_codec_spec &s, int mode, bool canon_pending) {
  if (mode == CC_NAIVE) return 0;
  if (s.codec == CC_TOPK && canon_pending) return 2;
  return 1;
}

}  // namespace
}  // namespace cc

using namespace cc;

struct cc_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  bool owned = false;
};

struct cc_allgather_layer {
  cc_comm *c = nullptr;
  cc_codec_spec spec{};
  int mode = CC_WITH_FEEDBACK, warmup = 1, x_dtype = CC_BF16;
  int64_t rows = 0, cols = 0, lo = 0, hi = 0;
  std::vector<int64_t> lo_of, hi_of;
  float *full = nullptr, *aux = nullptr, *loop = nullptr;
  uint8_t *sendbuf = nullptr, *recvbuf = nullptr, *ws = nullptr;
  int64_t slot = 0, ws_bytes = 0;
  double *record = nullptr;
  void *reg_send = nullptr, *reg_recv = nullptr;
  int step = 0;
  bool canon_pending = true;
  int64_t last_body = 0, last_wire = 0;
};

struct cc_alltoall_layer {
  cc_comm *c = nullptr;
  cc_codec_spec spec{};
  int mode = CC_WITH_FEEDBACK, warmup = 1, x_dtype = CC_BF16;
  int64_t n = 0, C = 0, cw = 0;
  float *base = nullptr, *aux = nullptr, *out = nullptr;
  uint8_t *sendbuf = nullptr, *recvbuf = nullptr, *ws = nullptr;
  int64_t slot = 0, ws_bytes = 0;
  double *record = nullptr;
  int step = 0;
  bool canon_pending = true;
};

extern "C" {

CC_API int cc_comm_get_unique_id(uint8_t *id_out) {
  if (int rc = need_nccl()) return rc;
  if (!id_out) {
    set_error("null id buffer");
    return CC_ERR_ARG;
  }
  ncclUniqueId id;
  if (int rc = nccl_status(nccl().GetUniqueId(&id), "ncclGetUniqueId")) return rc;
  std::memcpy(id_out, id.internal, sizeof(id.internal));
  return CC_OK;
}

CC_API int cc_comm_init_rank(const uint8_t *id, int nranks, int rank, cc_comm **out) {
  if (int rc = need_nccl()) return rc;
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("bad comm init arguments");
    return CC_ERR_ARG;
  }
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  ncclComm_t comm;
  if (int rc = nccl_status(nccl().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank")) return rc;
  auto *c = new cc_comm;
  c->comm = comm;
  c->rank = rank;
  c->nranks = nranks;
  c->owned = true;
  *out = c;
  return CC_OK;
}

CC_API int cc_comm_wrap(void *nccl_comm, cc_comm **out) {
  if (int rc = need_nccl()) return rc;
  if (!nccl_comm || !out) {
    set_error("null communicator");
    return CC_ERR_ARG;
  }
  auto *c = new cc_comm;
  c->comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  if (int rc = nccl_status(nccl().CommCount(c->comm, &c->nranks), "ncclCommCount")) {
    delete c;
    return rc;
  }
  if (int rc = nccl_status(nccl().CommUserRank(c->comm, &c->rank), "ncclCommUserRank")) {
    delete c;
    return rc;
  }
  *out = c;
  return CC_OK;
}

CC_API int cc_comm_rank(const cc_comm *c) { return c ? c->rank : CC_ERR_ARG; }
CC_API int cc_comm_size(const cc_comm *c) { return c ? c->nranks : CC_ERR_ARG; }

CC_API int cc_comm_destroy(cc_comm *c) {
  if (!c) return CC_OK;
  int rc = CC_OK;
  if (c->owned && c->comm) rc = nccl_status(nccl().CommDestroy(c->comm), "ncclCommDestroy");
  delete c;
  return rc;
}

// ---------------------------------------------------------------------------
// patch parallelism: compressed all-gather of row shards (mesh:188-237)
// ---------------------------------------------------------------------------

CC_API int cc_allgather_destroy(cc_allgather_layer *L) {
  if (!L) return CC_OK;
  if (L->c && nccl().ok && nccl().CommDeregister) {
    if (L->reg_send) nccl().CommDeregister(L->c->comm, L->reg_send);
    if (L->reg_recv) nccl().CommDeregister(L->c->comm, L->reg_recv);
  }
  cudaFree(L->full);
  cudaFree(L->aux);
  cudaFree(L->loop);
  cudaFree(L->sendbuf);
  cudaFree(L->recvbuf);
  cudaFree(L->ws);
  cudaFree(L->record);
  delete L;
  return CC_OK;
}

CC_API int cc_allgather_create(cc_comm *c, const cc_codec_spec *spec, int mode, int64_t rows, int64_t cols,
                               int warmup, int x_dtype, cc_allgather_layer **out) {
  if (int rc = check_spec(spec)) return rc;
  if (!out || (mode != CC_NAIVE && mode != CC_NO_FEEDBACK && mode != CC_WITH_FEEDBACK) || warmup < 1 ||
      (x_dtype != CC_F32 && x_dtype != CC_BF16)) {
    set_error("bad all-gather layer arguments");
    return CC_ERR_ARG;
  }
  const int P = c ? c->nranks : 1, rank = c ? c->rank : 0;
  if (rows < P || cols < 1) {
    set_error("cannot shard rows across ranks");
    return CC_ERR_SHAPE;
  }
  auto *L = new cc_allgather_layer;
  L->c = c;
  L->spec = *spec;
  L->mode = mode;
  L->warmup = warmup;
  L->x_dtype = x_dtype;
  L->rows = rows;
  L->cols = cols;
  const int64_t q = rows / P;  // contiguous shards, the last takes the remainder (mesh:125-135)
  int64_t max_rows = 0, max_body = 0;
  for (int d = 0; d < P; ++d) {
    L->lo_of.push_back(d * q);
    L->hi_of.push_back(d == P - 1 ? rows : (d + 1) * q);
    const int64_t r = L->hi_of.back() - L->lo_of.back();
    max_rows = std::max(max_rows, r);
    if (spec->codec != CC_RAW) max_body = std::max(max_body, body_of(*spec, r, cols));
  }
  L->lo = L->lo_of[rank];
  L->hi = L->hi_of[rank];
  const int64_t esz = x_dtype == CC_BF16 ? 2 : 4;
  L->slot = (std::max(max_body, max_rows * cols * esz) + 255) / 256 * 256;
  const int64_t own = L->hi - L->lo;
  L->ws_bytes = ws_of(*spec, own, cols);
  int rc = CC_OK;
  if (!rc) rc = dalloc(&L->full, sizeof(float) * rows * cols);
  if (!rc && mode != CC_NAIVE) rc = dalloc(&L->aux, sizeof(float) * own * cols);
  if (!rc && P == 1) rc = dalloc(&L->loop, sizeof(float) * rows * cols);
  if (!rc) rc = dalloc(&L->sendbuf, (size_t)L->slot);
  if (!rc && P > 1) rc = dalloc(&L->recvbuf, (size_t)L->slot * P);
  if (!rc) rc = dalloc(&L->ws, (size_t)std::max<int64_t>(L->ws_bytes, 256));
  if (!rc) rc = dalloc(&L->record, 2 * sizeof(double));
  if (rc) {
    cc_allgather_destroy(L);
    return rc;
  }
  if (P > 1 && nccl().CommRegister) {  // best effort: registered user buffers
    if (nccl().CommRegister(c->comm, L->sendbuf, (size_t)L->slot, &L->reg_send) != ncclSuccess) L->reg_send = nullptr;
    if (nccl().CommRegister(c->comm, L->recvbuf, (size_t)L->slot * P, &L->reg_recv) != ncclSuccess)
      L->reg_recv = nullptr;
  }
  *out = L;
  return CC_OK;
}

CC_API int cc_allgather_step(cc_allgather_layer *L, const void *x_shard, void *stream) {
  if (!L || !x_shard) {
    set_error("null layer / input");
    return CC_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int P = L->c ? L->c->nranks : 1, rank = L->c ? L->c->rank : 0;
  const int64_t C = L->cols, own = L->hi - L->lo;
  const int t = L->step + 1;
  const cc_codec_spec &s = L->spec;
  const bool warm = t <= L->warmup || s.codec == CC_RAW;  // warmup / identity send raw (pl:89-97)
  float *base = L->full + L->lo * C;
  // ---- encode own shard (pl:84-121) straight into the send buffer ----
  int rc;
  int64_t nbytes;
  if (warm) {
    nbytes = own * C * (L->x_dtype == CC_BF16 ? 2 : 4);
    rc = cc_warmup_step(L->mode, own, C, x_shard, L->x_dtype, base, L->aux, L->sendbuf, L->x_dtype, L->record, stream);
  } else if (quant(s.codec)) {
    nbytes = body_of(s, own, C);
    rc = cc_encode_step(s.codec, L->mode, s.scale_mode, own, C, x_shard, L->x_dtype, base, L->aux, L->sendbuf, L->ws,
                        L->ws_bytes, L->record, stream);
  } else if (s.codec == CC_TOPK) {
    nbytes = body_of(s, own, C);
    rc = cc_topk_encode_step(L->mode, own, C, param_of(s, own, C), x_shard, L->x_dtype, base, L->aux, L->sendbuf, L->ws,
                             L->ws_bytes, L->record, stream);
  } else {
    nbytes = body_of(s, own, C);
    rc = cc_nm_encode_step(L->mode, own, C, s.nm_n, s.nm_m, x_shard, L->x_dtype, base, L->aux, L->sendbuf, L->ws,
                           L->ws_bytes, L->record, stream);
  }
  if (rc) return rc;
  // ---- equal-size collective of the bodies (every rank sends the largest shard's size) ----
  int64_t per = 0;
  for (int d = 0; d < P; ++d) {
    const int64_t r = L->hi_of[d] - L->lo_of[d];
    per = std::max(per, warm ? r * C * (L->x_dtype == CC_BF16 ? 2 : 4) : body_of(s, r, C));
  }
  per = (per + 15) / 16 * 16;  // aligned receive slots for the vectorised decoders
  L->last_body = nbytes;
  L->last_wire = per;
  const int acc = (warm) ? 0 : receiver_acc(s, L->mode, L->canon_pending);
  const int tag = warm ? CC_RAW : s.codec;
  const int dt = warm ? L->x_dtype : CC_F32;
  if (P == 1) {  // world 1: loopback receiver (BASELINE config 1, pl:182-192)
    const int64_t param = warm ? 0 : param_of(s, L->rows, C);
    rc = cc_decode_step(tag, acc, L->rows, C, param, L->sendbuf, dt, L->loop, stream);
  } else {
    if (int r2 = need_nccl()) return r2;
    rc = nccl_status(nccl().AllGather(L->sendbuf, L->recvbuf, (size_t)per, ncclUint8, L->c->comm, st), "ncclAllGather");
    if (rc) return rc;
    // ---- decode every peer into its rows of the reconstruction (mesh:232-236) ----
    std::vector<int64_t> rows;
    std::vector<const uint8_t *> bodies;
    std::vector<float *> bases;
    bool uneven = false;
    for (int d = 0; d < P; ++d) {
      if (d == rank) continue;
      rows.push_back(L->hi_of[d] - L->lo_of[d]);
      bodies.push_back(L->recvbuf + (size_t)d * per);
      bases.push_back(L->full + L->lo_of[d] * C);
      uneven |= rows.back() != rows.front();
    }
    if (!warm && s.codec == CC_TOPK && uneven) {  // k depends on the shard height
      for (size_t i = 0; i < rows.size() && !rc; ++i)
        rc = cc_decode_step(tag, acc, rows[i], C, param_of(s, rows[i], C), bodies[i], dt, bases[i], stream);
    } else {
      const int64_t param = warm ? 0 : param_of(s, rows.front(), C);
      rc = cc_decode_batched(tag, acc, (int)rows.size(), rows.data(), C, param, bodies.data(), dt, bases.data(),
                             stream);
    }
  }
  if (rc) return rc;
  L->canon_pending = warm || (L->canon_pending && acc == 0);
  L->step = t;
  return CC_OK;
}

CC_API float *cc_allgather_reconstruction(cc_allgather_layer *L) {
  if (!L) return nullptr;
  return (L->c && L->c->nranks > 1) ? L->full : L->loop;
}
CC_API float *cc_allgather_sender_base(cc_allgather_layer *L) { return L ? L->full + L->lo * L->cols : nullptr; }
CC_API float *cc_allgather_sender_aux(cc_allgather_layer *L) { return L ? L->aux : nullptr; }
CC_API const uint8_t *cc_allgather_body(cc_allgather_layer *L, int64_t *nbytes) {
  if (!L) return nullptr;
  if (nbytes) *nbytes = L->last_body;
  return L->sendbuf;
}
CC_API const double *cc_allgather_record(cc_allgather_layer *L) { return L ? L->record : nullptr; }
CC_API int cc_allgather_shard(cc_allgather_layer *L, int64_t *lo, int64_t *hi) {
  if (!L) return CC_ERR_ARG;
  if (lo) *lo = L->lo;
  if (hi) *hi = L->hi;
  return CC_OK;
}

// ---------------------------------------------------------------------------
// Ulysses: compressed all-to-all, one channel per directed (src, dst) chunk
// (SPEC.md:473): rank r sends column chunk d of its [n, C] rows to rank d and
// rebuilds out[P n, C / P] (the full sequence for its heads).
// ---------------------------------------------------------------------------

CC_API int cc_alltoall_destroy(cc_alltoall_layer *L) {
  if (!L) return CC_OK;
  cudaFree(L->base);
  cudaFree(L->aux);
  cudaFree(L->out);
  cudaFree(L->sendbuf);
  cudaFree(L->recvbuf);
  cudaFree(L->ws);
  cudaFree(L->record);
  delete L;
  return CC_OK;
}

CC_API int cc_alltoall_create(cc_comm *c, const cc_codec_spec *spec, int mode, int64_t n_local, int64_t cols,
                              int warmup, int x_dtype, cc_alltoall_layer **out) {
  if (int rc = check_spec(spec)) return rc;
  if (!quant(spec->codec) && spec->codec != CC_RAW) {
    set_error("cc_alltoall: codecs sign1 / quant2 / quant4 / raw");
    return CC_ERR_UNSUPPORTED;
  }
  const int P = c ? c->nranks : 1;
  if (!out || n_local < 1 || cols < 1 || cols % P || warmup < 1 || (x_dtype != CC_F32 && x_dtype != CC_BF16) ||
      (mode != CC_NAIVE && mode != CC_NO_FEEDBACK && mode != CC_WITH_FEEDBACK)) {
    set_error("bad all-to-all layer arguments (cols must divide by the world size)");
    return CC_ERR_ARG;
  }
  auto *L = new cc_alltoall_layer;
  L->c = c;
  L->spec = *spec;
  L->mode = mode;
  L->warmup = warmup;
  L->x_dtype = x_dtype;
  L->n = n_local;
  L->C = cols;
  L->cw = cols / P;
  const int64_t esz = x_dtype == CC_BF16 ? 2 : 4;
  const int64_t body = spec->codec == CC_RAW ? 0 : body_of(*spec, n_local, L->cw);
  L->slot = (std::max(body, n_local * L->cw * esz) + 255) / 256 * 256;
  L->ws_bytes = spec->codec == CC_RAW ? 0 : cc_workspace_bytes(spec->codec, n_local, cols, 0);
  int rc = CC_OK;
  if (!rc) rc = dalloc(&L->base, sizeof(float) * n_local * cols);
  if (!rc && mode != CC_NAIVE) rc = dalloc(&L->aux, sizeof(float) * n_local * cols);
  if (!rc) rc = dalloc(&L->out, sizeof(float) * P * n_local * L->cw);
  if (!rc) rc = dalloc(&L->sendbuf, (size_t)L->slot * P);
  if (!rc) rc = dalloc(&L->recvbuf, (size_t)L->slot * P);
  if (!rc) rc = dalloc(&L->ws, (size_t)std::max<int64_t>(L->ws_bytes, 256));
  if (!rc) rc = dalloc(&L->record, 2 * sizeof(double) * P);
  if (rc) {
    cc_alltoall_destroy(L);
    return rc;
  }
  *out = L;
  return CC_OK;
}

CC_API int cc_alltoall_step(cc_alltoall_layer *L, const void *x_local, void *stream) {
  if (!L || !x_local) {
    set_error("null layer / input");
    return CC_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int P = L->c ? L->c->nranks : 1;
  const int64_t n = L->n, C = L->C, cw = L->cw;
  const int t = L->step + 1;
  const cc_codec_spec &s = L->spec;
  const bool warm = t <= L->warmup || s.codec == CC_RAW;
  const int64_t esz = L->x_dtype == CC_BF16 ? 2 : 4;
  int rc;
  int64_t per;
  if (warm) {
    // raw step on the full rows (pl:89-97), then each chunk's raw body (lossless bf16
    // for bf16 inputs) into its send slot
    uint8_t *tmp = L->recvbuf;  // free until the collective below
    rc = cc_warmup_step(L->mode, n, C, x_local, L->x_dtype, L->base, L->aux, tmp, L->x_dtype, L->record, stream);
    if (rc) return rc;
    per = n * cw * esz;
    for (int d = 0; d < P && !rc; ++d)
      if (cudaMemcpy2DAsync(L->sendbuf + (size_t)d * L->slot, (size_t)(cw * esz),
                            static_cast<const uint8_t *>(x_local) + (size_t)d * cw * esz, (size_t)(C * esz),
                            (size_t)(cw * esz), (size_t)n, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = cuda_status("chunk copy");
    if (rc) return rc;
  } else {
    rc = cc_encode_step_segmented(s.codec, L->mode, s.scale_mode, n, C, P, x_local, L->x_dtype, L->base, L->aux,
                                  L->sendbuf, L->slot, L->ws, L->ws_bytes, L->record, stream);
    if (rc) return rc;
    per = body_of(s, n, cw);
  }
  // ---- all-to-all: chunk d -> rank d; slot s of the receive buffer <- rank s ----
  if (P > 1) {
    if (int r2 = need_nccl()) return r2;
    if ((rc = nccl_status(nccl().GroupStart(), "ncclGroupStart"))) return rc;
    for (int d = 0; d < P && !rc; ++d) {
      rc = nccl_status(nccl().Send(L->sendbuf + (size_t)d * L->slot, (size_t)per, ncclUint8, d, L->c->comm, st),
                       "ncclSend");
      if (!rc)
        rc = nccl_status(nccl().Recv(L->recvbuf + (size_t)d * L->slot, (size_t)per, ncclUint8, d, L->c->comm, st),
                         "ncclRecv");
    }
    const int rc2 = nccl_status(nccl().GroupEnd(), "ncclGroupEnd");
    if (rc || rc2) return rc ? rc : rc2;
  } else if (cudaMemcpyAsync(L->recvbuf, L->sendbuf, (size_t)per, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    return cuda_status("loopback copy");
  }
  // ---- decode the P received chunks into out[s n : (s + 1) n] ----
  const int acc = warm ? 0 : receiver_acc(s, L->mode, L->canon_pending);
  std::vector<int64_t> rows(P, n);
  std::vector<const uint8_t *> bodies(P);
  std::vector<float *> bases(P);
  for (int d = 0; d < P; ++d) {
    bodies[d] = L->recvbuf + (size_t)d * L->slot;
    bases[d] = L->out + (size_t)d * n * cw;
  }
  rc = cc_decode_batched(warm ? CC_RAW : s.codec, acc, P, rows.data(), cw, 0, bodies.data(), warm ? L->x_dtype : CC_F32,
                         bases.data(), stream);
  if (rc) return rc;
  L->canon_pending = warm || (L->canon_pending && acc == 0);
  L->step = t;
  return CC_OK;
}

CC_API float *cc_alltoall_output(cc_alltoall_layer *L) { return L ? L->out : nullptr; }
CC_API float *cc_alltoall_sender_base(cc_alltoall_layer *L) { return L ? L->base : nullptr; }

}  // extern "C"
