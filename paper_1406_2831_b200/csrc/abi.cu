// Library-level C ABI: version, thread-local error string, launch counter,
// context lifetime.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ctx.cuh"

namespace krb {

static thread_local char g_err[1024] = "";
static int64_t g_launches = 0;

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int64_t &launch_counter() { return g_launches; }

static krb_alloc_fn g_alloc = nullptr;
static krb_free_fn g_free = nullptr;
static bool g_allocated = false;   // any dev_alloc yet (the hook is fixed after)

cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t st) {
  g_allocated = true;
  if (g_alloc) {
    *p = g_alloc(bytes ? bytes : 8, (void *)st);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMallocAsync(p, bytes, st);
}

void dev_free(void *p, cudaStream_t st) {
  if (!p) return;
  if (g_free)
    g_free(p, (void *)st);
  else if (st)
    cudaFreeAsync(p, st);
  else
    cudaFree(p);
}

Tuning &tuning() {
  static Tuning t;
  return t;
}

}  // namespace krb

extern "C" {

int krb_abi_version(void) { return 1; }

const char *krb_last_error(void) { return krb::g_err; }

int64_t krb_launch_count(void) { return krb::g_launches; }

int krb_set_tuning(const char *key, int64_t value) {
  KRB_REQUIRE(key != nullptr, "krb_set_tuning: NULL key");
  krb::Tuning &t = krb::tuning();
  struct { const char *name; int *slot; } table[] = {
      {"persist0", &t.persist0},   {"p0_grid_half", &t.p0_grid_half},
      {"p0_onchip", &t.p0_onchip}, {"p0_prof_cta", &t.p0_prof_cta},
      {"cluster", &t.cluster},     {"persist_v1", &t.persist_v1},
      {"gemm_mode", &t.gemm_mode}, {"l2keep", &t.l2keep},
      {"phase_variant", &t.phase_variant}, {"tdot_variant", &t.tdot_variant},
      {"spmv_variant", &t.spmv_variant}, {"spmv_prefetch_mb", &t.spmv_prefetch_mb},
      {"spmm_variant", &t.spmm_variant}, {"phase_pf_rows", &t.phase_pf_rows},
      {"value_coding", &t.value_coding}};
  for (auto &e : table)
    if (strcmp(e.name, key) == 0) {
      *e.slot = (int)value;
      return KRB_OK;
    }
  krb::set_error("krb_set_tuning: unknown key '%s'", key);
  return KRB_EINVAL;
}

int krb_set_allocator(krb_alloc_fn alloc, krb_free_fn free_fn) {
  KRB_REQUIRE((alloc == nullptr) == (free_fn == nullptr),
              "krb_set_allocator: give both functions or neither");
  if (krb::g_alloc == alloc && krb::g_free == free_fn) return KRB_OK;
  KRB_REQUIRE(!krb::g_allocated,
              "krb_set_allocator: device memory was already allocated");
  krb::g_alloc = alloc;
  krb::g_free = free_fn;
  return KRB_OK;
}

int krb_reset_tuning(void) {
  krb::tuning() = krb::Tuning();
  return KRB_OK;
}

int krb_memcpy_d2d(void *d_dst, const void *d_src, int64_t bytes, void *stream) {
  KRB_REQUIRE(bytes >= 0, "krb_memcpy_d2d: negative size");
  if (bytes == 0) return KRB_OK;
  KRB_CHECK_CUDA(cudaMemcpyAsync(d_dst, d_src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                 krb::as_stream(stream)));
  return KRB_OK;
}

int krb_context_create(krb_context **out) {
  KRB_REQUIRE(out != nullptr, "krb_context_create: out is NULL");
  *out = new krb_context();
  return KRB_OK;
}

int krb_context_destroy(krb_context *ctx) {
  if (!ctx) return KRB_OK;
  ctx->graph.reset();
  krb::rbicg_cache_free(ctx);
  krb::batch_pool_free(ctx);
  double *bufs[] = {ctx->part, ctx->x, ctx->r, ctx->p, ctx->q, ctx->s,
                    ctx->t, ctx->rt0, ctx->b, ctx->w, ctx->p2, ctx->q2, ctx->kbuf};
  for (double *b : bufs)
    if (b) cudaFree(b);
  if (ctx->S) cudaFree(ctx->S);
  if (ctx->desc) cudaFree(ctx->desc);
  if (ctx->counters) cudaFree(ctx->counters);
  delete ctx;
  return KRB_OK;
}

}  // extern "C"
