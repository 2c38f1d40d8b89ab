// capi.cu -- the extern "C" boundary of libosmpm (include/osmpm.h): argument checking, dispatch on
// (dimension, precision), error strings.  No compute happens here.
#include <cstdio>
#include <cstring>
#include <string>

#include "coupler.cuh"
#include "transmit.cuh"
#include "dist.cuh"

namespace osmpm {

static thread_local std::string g_err;

void set_error(const char* fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}
void prefix_error(const char* fmt, ...)
{
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = std::string(buf) + g_err;
}

cudaEvent_t Profiler::begin(const std::string& name, cudaStream_t s)
{
    Fam& f = fams[name];
    if (f.used == f.ev.size()) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        f.ev.push_back({a, b});
    }
    cudaEventRecord(f.ev[f.used].first, s);
    return f.ev[f.used].first;
}

void Profiler::end(const std::string& name, cudaStream_t s)
{
    Fam& f = fams[name];
    cudaEventRecord(f.ev[f.used].second, s);
    f.used++;
}

osmpm_status Profiler::query(const std::string& name, int64_t* launches, double* ms)
{
    *launches = 0;
    *ms = 0.0;
    auto it = fams.find(name);
    if (it == fams.end()) return OSMPM_OK;
    double tot = 0.0;
    for (size_t i = 0; i < it->second.used; ++i) {
        float t = 0.f;
        OSMPM_CU(cudaEventSynchronize(it->second.ev[i].second));
        OSMPM_CU(cudaEventElapsedTime(&t, it->second.ev[i].first, it->second.ev[i].second));
        tot += t;
    }
    *launches = (int64_t)it->second.used;
    *ms = tot;
    return OSMPM_OK;
}

void Profiler::reset()
{
    for (auto& kv : fams) kv.second.used = 0;
}

Profiler::~Profiler()
{
    for (auto& kv : fams)
        for (auto& e : kv.second.ev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
}

// CUDA-core FMA throughput probe (the FP64 / FP32 vector peaks are not in
// MEASURED_PEAKS.json): every thread runs 8 independent FMA chains of `iters` steps on registers
template <typename T>
__global__ void __launch_bounds__(256) k_fma_probe(int iters, T a, T b, T* out)
{
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k) * (T)1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == (T)-1.2345) out[0] = s;  // never true: keeps the chains alive
}

}  // namespace osmpm

using namespace osmpm;

#define CHECK_ARG(cond, ...)                                                                        \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            set_error(__VA_ARGS__);                                                                 \
            return OSMPM_E_INVALID_ARG;                                                             \
        }                                                                                           \
    } while (0)

#define SET_DEVICE(ctx) OSMPM_CU(cudaSetDevice((ctx)->device))

extern "C" {

const char* osmpm_last_error(void) { return g_err.c_str(); }
#ifndef OSMPM_SRC_HASH
#define OSMPM_SRC_HASH "unknown"
#endif
const char* osmpm_version(void) { return "osmpm 0.2 (sm_100a) src " OSMPM_SRC_HASH; }

osmpm_status osmpm_ctx_create(int device, void* cuda_stream, osmpm_ctx** out)
{
    CHECK_ARG(out, "out is NULL");
    osmpm_ctx* c = new osmpm_ctx();
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        set_error("cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
        delete c;
        return OSMPM_E_CUDA;
    }
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        c->own_stream = true;
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    *out = c;
    return OSMPM_OK;
}

void osmpm_ctx_destroy(osmpm_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->gc.comm) ncclCommDestroy(ctx->gc.comm);
    for (void* p : ctx->scratch)
        if (p) cudaFree(p);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

osmpm_status osmpm_profile_enable(osmpm_ctx* ctx, int enable)
{
    CHECK_ARG(ctx, "ctx is NULL");
    ctx->prof.on = enable != 0;
    return OSMPM_OK;
}
osmpm_status osmpm_profile_reset(osmpm_ctx* ctx)
{
    CHECK_ARG(ctx, "ctx is NULL");
    SET_DEVICE(ctx);
    OSMPM_CU(cudaStreamSynchronize(ctx->stream));
    ctx->prof.reset();
    return OSMPM_OK;
}
osmpm_status osmpm_kernel_time(osmpm_ctx* ctx, const char* family, int64_t* launches, double* ms)
{
    CHECK_ARG(ctx && family && launches && ms, "NULL argument");
    SET_DEVICE(ctx);
    return ctx->prof.query(family, launches, ms);
}

osmpm_status osmpm_launch_count(osmpm_ctx* ctx, int64_t* launches)
{
    CHECK_ARG(ctx && launches, "NULL argument");
    *launches = ctx->launches;
    return OSMPM_OK;
}

osmpm_status osmpm_comm_unique_id(uint8_t id[128])
{
    CHECK_ARG(id, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    OSMPM_NCCL(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
    return OSMPM_OK;
}

osmpm_status osmpm_ctx_init_comm(osmpm_ctx* ctx, int rank, int nranks, const uint8_t id[128])
{
    CHECK_ARG(ctx && id, "NULL argument");
    CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "rank %d / nranks %d invalid", rank, nranks);
    CHECK_ARG(!ctx->gc.comm, "communicator already initialised");
    SET_DEVICE(ctx);
    ctx->gc.rank = rank;
    ctx->gc.nranks = nranks;
    // a communicator of one rank too: the subdomains of this ctx then take the multi-rank code path
    // (NCCL all-reduces, all-gather, broadcast; neighbour exchanges find no neighbour), which is how
    // the NCCL calls run on a one-GPU box (tests/test_gpu_nccl1.py)
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    OSMPM_NCCL(ncclCommInitRank(&ctx->gc.comm, nranks, u, rank));
    return OSMPM_OK;
}

osmpm_status osmpm_slab_cuts(const int32_t* base_x, int64_t n, int32_t nslab, int32_t tile, int32_t* cuts)
{
    CHECK_ARG(nslab >= 1 && tile >= 1 && n >= 0 && (n == 0 || base_x) && (nslab == 1 || cuts), "bad arguments");
    std::vector<int> bx(base_x, base_x + n);
    std::vector<int> c = balanced_cuts(bx, nslab, tile);
    if ((int)c.size() != nslab - 1) {
        set_error("cannot cut %d slabs of %d-cell columns from %lld particles", nslab, tile, (long long)n);
        return OSMPM_E_INVALID_ARG;
    }
    for (int k = 0; k + 1 < nslab; ++k) cuts[k] = c[k];
    return OSMPM_OK;
}

osmpm_status osmpm_ctx_set_local_slabs(osmpm_ctx* ctx, int n)
{
    CHECK_ARG(ctx, "ctx is NULL");
    CHECK_ARG(n >= 1 && n <= 64, "local slabs %d outside [1, 64]", n);
    ctx->gc.local_slabs = n;
    return OSMPM_OK;
}

osmpm_status osmpm_subdomain_create(osmpm_ctx* ctx, const osmpm_grid_desc* grid, double dt,
                                    const osmpm_particles_view* particles, const osmpm_material* mats,
                                    int32_t n_mats, const double gravity[3], osmpm_precision prec,
                                    osmpm_subdomain** out)
{
    return osmpm_subdomain_create_ex(ctx, grid, dt, particles, mats, n_mats, gravity, prec, 1, out);
}

osmpm_status osmpm_subdomain_create_ex(osmpm_ctx* ctx, const osmpm_grid_desc* grid, double dt,
                                       const osmpm_particles_view* particles, const osmpm_material* mats,
                                       int32_t n_mats, const double gravity[3], osmpm_precision prec,
                                       int32_t decompose, osmpm_subdomain** out)
{
    CHECK_ARG(ctx && grid && particles && mats && out, "NULL argument");
    CHECK_ARG(grid->dim == 2 || grid->dim == 3, "dim = %d (must be 2 or 3)", grid->dim);
    CHECK_ARG(grid->dx > 0, "dx must be > 0");
    CHECK_ARG(dt > 0, "dt must be > 0");
    CHECK_ARG(particles->n >= 0 && particles->n < (int64_t(1) << 31), "n = %lld out of range",
              (long long)particles->n);
    CHECK_ARG(particles->n == 0 || (particles->x && particles->m && particles->V0), "x, m and V0 are required");
    for (int a = 0; a < grid->dim; ++a)
        CHECK_ARG(grid->dims[a] >= 3 && grid->dims[a] < (int64_t(1) << 30), "dims[%d] = %lld out of range", a,
                  (long long)grid->dims[a]);
    CHECK_ARG(prec == OSMPM_F64 || prec == OSMPM_F32, "bad precision");
    SET_DEVICE(ctx);
    osmpm_subdomain* s = nullptr;
    osmpm_status rc;
    const bool dist = decompose && (ctx->gc.multi() || ctx->gc.local_slabs > 1);
#define MAKE(DD, RR)                                                                                \
    if (dist) {                                                                                     \
        auto* q = new Dist<DD, RR>();                                                               \
        q->ctx = ctx;                                                                               \
        q->dim = DD;                                                                                \
        q->prec = prec;                                                                             \
        q->decomposed = true;                                                                       \
        s = q;                                                                                      \
        rc = q->create(grid, dt, particles, mats, n_mats, gravity);                                 \
    } else {                                                                                        \
        auto* q = new Sub<DD, RR>();                                                                \
        q->ctx = ctx;                                                                               \
        q->dim = DD;                                                                                \
        q->prec = prec;                                                                             \
        s = q;                                                                                      \
        rc = q->create(grid, dt, particles, mats, n_mats, gravity);                                 \
    }
    if (grid->dim == 3 && prec == OSMPM_F64) MAKE(3, double)
    else if (grid->dim == 2 && prec == OSMPM_F64) MAKE(2, double)
    else if (grid->dim == 3) MAKE(3, float)
    else MAKE(2, float)
#undef MAKE
    if (rc != OSMPM_OK) {
        delete s;
        return rc;
    }
    *out = s;
    return OSMPM_OK;
}

void osmpm_subdomain_destroy(osmpm_subdomain* sub)
{
    if (!sub) return;
    cudaSetDevice(sub->ctx->device);
    cudaStreamSynchronize(sub->ctx->stream);
    delete sub;
}

#define SUB_CALL(sub, expr)                                                                         \
    do {                                                                                            \
        CHECK_ARG(sub, "subdomain is NULL");                                                        \
        SET_DEVICE((sub)->ctx);                                                                     \
        return (sub)->expr;                                                                         \
    } while (0)

osmpm_status osmpm_set_gravity(osmpm_subdomain* sub, const double gravity[3])
{
    CHECK_ARG(gravity, "gravity is NULL");
    SUB_CALL(sub, set_gravity(gravity));
}
osmpm_status osmpm_set_dt(osmpm_subdomain* sub, double dt) { SUB_CALL(sub, set_dt(dt)); }
osmpm_status osmpm_set_particles(osmpm_subdomain* sub, const double* x, const double* v, const double* F,
                                 const double* B, osmpm_memspace space)
{
    SUB_CALL(sub, set_particles(x, v, F, B, space));
}
osmpm_status osmpm_set_dirichlet(osmpm_subdomain* sub, int64_t n, const int64_t* node_idx, const uint8_t* comp_mask,
                                 const double* vel, osmpm_memspace space)
{
    CHECK_ARG(n >= 0 && (n == 0 || (node_idx && comp_mask && vel)), "bad Dirichlet arguments");
    SUB_CALL(sub, set_dirichlet(n, node_idx, comp_mask, vel, space));
}
osmpm_status osmpm_p2g(osmpm_subdomain* sub) { SUB_CALL(sub, p2g()); }
osmpm_status osmpm_read_grid(osmpm_subdomain* sub, double* m, double* p, double* v, double* f_ext, double* f_sigma,
                             uint8_t* active, osmpm_memspace space)
{
    SUB_CALL(sub, read_grid(m, p, v, f_ext, f_sigma, active, space));
}
osmpm_status osmpm_newton_gradient(osmpm_subdomain* sub, const double* u, double* g, double* E, osmpm_memspace space)
{
    CHECK_ARG(u, "u is NULL");
    SUB_CALL(sub, newton_gradient(u, g, E, space));
}
osmpm_status osmpm_newton_hvp(osmpm_subdomain* sub, const double* d, double* y, osmpm_memspace space)
{
    CHECK_ARG(d && y, "d / y is NULL");
    SUB_CALL(sub, newton_hvp(d, y, space));
}
osmpm_status osmpm_newton_diag(osmpm_subdomain* sub, double* diag, osmpm_memspace space)
{
    CHECK_ARG(diag, "diag is NULL");
    SUB_CALL(sub, newton_diag(diag, space));
}
osmpm_status osmpm_implicit_solve(osmpm_subdomain* sub, const osmpm_newton_settings* settings,
                                  osmpm_solve_stats* stats)
{
    CHECK_ARG(settings, "settings is NULL");
    CHECK_ARG(settings->max_newton >= 0 && settings->max_cg >= 0, "negative iteration caps");
    CHECK_ARG(settings->cg_variant == 0 || settings->cg_variant == 1, "cg_variant must be 0 or 1");
    CHECK_ARG(settings->psd >= 0 && settings->psd <= 2, "psd must be 0, 1 or 2");
    SUB_CALL(sub, implicit_solve(settings, stats));
}
osmpm_status osmpm_read_grid_velocity(osmpm_subdomain* sub, double* v, osmpm_memspace space)
{
    CHECK_ARG(v, "v is NULL");
    SUB_CALL(sub, read_grid_velocity(v, space));
}
osmpm_status osmpm_set_grid_velocity(osmpm_subdomain* sub, const double* v, osmpm_memspace space)
{
    CHECK_ARG(v, "v is NULL");
    SUB_CALL(sub, set_grid_velocity(v, space));
}
osmpm_status osmpm_g2p(osmpm_subdomain* sub) { SUB_CALL(sub, g2p()); }
osmpm_status osmpm_read_particles(osmpm_subdomain* sub, double* x, double* v, double* F, double* B,
                                  osmpm_memspace space)
{
    SUB_CALL(sub, read_particles(x, v, F, B, space));
}
osmpm_status osmpm_subdomain_info(osmpm_subdomain* sub, int64_t* n_particles, int64_t box_lo[3], int64_t box_dims[3])
{
    SUB_CALL(sub, info(n_particles, box_lo, box_dims));
}
osmpm_status osmpm_sync(osmpm_subdomain* sub) { SUB_CALL(sub, sync()); }
osmpm_status osmpm_sort_pairs(osmpm_ctx* ctx, uint32_t* keys, int32_t* vals, int64_t n, int32_t nbits,
                              osmpm_memspace space)
{
    CHECK_ARG(ctx, "ctx is NULL");
    CHECK_ARG(n >= 0 && n < (int64_t(1) << 31), "n outside [0, 2^31)");
    CHECK_ARG(nbits >= 0 && nbits <= 32, "nbits outside [0, 32]");
    CHECK_ARG(n == 0 || (keys && vals), "NULL keys / vals");
    SET_DEVICE(ctx);
    if (n == 0 || nbits == 0) return OSMPM_OK;
    DBuf<uint32_t> k[2], h;
    DBuf<int> v[2];
    for (int i = 0; i < 2; ++i) {
        OSMPM_TRY(k[i].need(n));
        OSMPM_TRY(v[i].need(n));
    }
    OSMPM_TRY(h.need(radix_hist_words(n)));
    const cudaMemcpyKind in = space == OSMPM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind out = space == OSMPM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    OSMPM_CU(cudaMemcpyAsync(k[0].p, keys, n * 4, in, ctx->stream));
    OSMPM_CU(cudaMemcpyAsync(v[0].p, vals, n * 4, in, ctx->stream));
    const int r = radix_sort_pairs(k[0].p, v[0].p, k[1].p, v[1].p, n, nbits, h.p, ctx->stream, ctx->launches) ? 1 : 0;
    OSMPM_LAUNCH_CHECK();
    OSMPM_CU(cudaMemcpyAsync(keys, k[r].p, n * 4, out, ctx->stream));
    OSMPM_CU(cudaMemcpyAsync(vals, v[r].p, n * 4, out, ctx->stream));
    OSMPM_CU(cudaStreamSynchronize(ctx->stream));
    return OSMPM_OK;
}
osmpm_status osmpm_measure_fma_peak(osmpm_ctx* ctx, osmpm_precision prec, double* tflops)
{
    CHECK_ARG(ctx && tflops, "NULL argument");
    SET_DEVICE(ctx);
    int sms = 0;
    OSMPM_CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    DBuf<double> out;
    OSMPM_TRY(out.need(1));
    cudaEvent_t e0, e1;
    OSMPM_CU(cudaEventCreate(&e0));
    OSMPM_CU(cudaEventCreate(&e1));
    auto launch = [&]() {
        if (prec == OSMPM_F64)
            k_fma_probe<double><<<blocks, threads, 0, ctx->stream>>>(iters, 0.999999, 1e-7, out.p);
        else
            k_fma_probe<float><<<blocks, threads, 0, ctx->stream>>>(iters, 0.999999f, 1e-7f, (float*)out.p);
        ctx->launches++;
    };
    launch();  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        OSMPM_CU(cudaEventRecord(e0, ctx->stream));
        launch();
        OSMPM_CU(cudaEventRecord(e1, ctx->stream));
        OSMPM_CU(cudaEventSynchronize(e1));
        float ms = 0.f;
        OSMPM_CU(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    OSMPM_LAUNCH_CHECK();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    return OSMPM_OK;
}

osmpm_status osmpm_checkpoint(osmpm_subdomain* sub) { SUB_CALL(sub, checkpoint()); }
osmpm_status osmpm_restore(osmpm_subdomain* sub) { SUB_CALL(sub, restore()); }

osmpm_status osmpm_subdomain_decomp(osmpm_subdomain* sub, int32_t* slabs_total, int32_t* slabs_local,
                                    int32_t* first_slab, int64_t* n_local, int32_t* cuts)
{
    CHECK_ARG(sub, "subdomain is NULL");
    SET_DEVICE(sub->ctx);
    int32_t st = 1, sl = 1, fs = 0;
    std::vector<int> cv;
#define DEC(DD, RR)                                                                                 \
    if (sub->dim == DD && sub->prec == (sizeof(RR) == 8 ? OSMPM_F64 : OSMPM_F32)) {                 \
        auto* d = static_cast<Dist<DD, RR>*>(sub);                                                  \
        st = d->nslab_total;                                                                        \
        sl = (int32_t)d->sp.size();                                                                 \
        fs = d->first_slab;                                                                         \
        cv = d->cuts;                                                                               \
    }
    if (sub->decomposed) {
        DEC(3, double) DEC(2, double) DEC(3, float) DEC(2, float)
    }
#undef DEC
    if (slabs_total) *slabs_total = st;
    if (slabs_local) *slabs_local = sl;
    if (first_slab) *first_slab = fs;
    if (cuts)
        for (size_t k = 0; k < cv.size(); ++k) cuts[k] = cv[k];
    if (n_local) return sub->info(n_local, nullptr, nullptr);
    return OSMPM_OK;
}

osmpm_status osmpm_transmit(osmpm_subdomain* src, osmpm_subdomain* dst, osmpm_direction dir, double alpha,
                            double eps_tol, int64_t n_targets, const int64_t* targets, double* v_out,
                            osmpm_memspace space)
{
    CHECK_ARG(src && dst && v_out, "NULL argument");
    CHECK_ARG(src->dim == dst->dim && src->prec == dst->prec, "transmit: subdomains differ in dim / precision");
    CHECK_ARG(src->ctx == dst->ctx, "transmit: subdomains belong to different contexts");
    CHECK_ARG(n_targets >= 0, "n_targets < 0");
    SET_DEVICE(src->ctx);
#define TR(DD, RR)                                                                                  \
    {                                                                                               \
        using SubT = Sub<DD, RR>;                                                                   \
        using DistT = Dist<DD, RR>;                                                                 \
        SubT* s_sub = src->decomposed ? nullptr : static_cast<SubT*>(src);                          \
        SubT* d_sub = dst->decomposed ? nullptr : static_cast<SubT*>(dst);                          \
        SlabGroup<DD, RR> SG = src->decomposed ? static_cast<DistT*>(src)->group() : s_sub->self_group(); \
        GridGeo geo = dst->decomposed ? geo_of(static_cast<DistT*>(dst)) : geo_of(d_sub);           \
        const int64_t dn = dst->decomposed ? static_cast<DistT*>(dst)->dense_nodes() : d_sub->dense_nodes(); \
        return transmit_impl<DD, RR>(SG, s_sub, d_sub, geo, dn, dir, alpha, eps_tol, n_targets, targets, v_out, \
                                     space);                                                        \
    }
    if (src->dim == 3 && src->prec == OSMPM_F64) TR(3, double);
    if (src->dim == 2 && src->prec == OSMPM_F64) TR(2, double);
    if (src->dim == 3) TR(3, float);
    TR(2, float);
#undef TR
}

osmpm_status osmpm_schwarz_receivers_host(const osmpm_grid_desc* coarse, const int64_t coarse_lo[3],
                                          const int64_t coarse_dims[3], const double* m_b, const uint8_t* gamma_b,
                                          const uint8_t* active_b, const osmpm_grid_desc* fine,
                                          const int64_t fine_lo[3], const int64_t fine_dims[3], int64_t nown,
                                          const double* m_s, const double* mb_s, const uint8_t* active_s,
                                          double tau_s, uint8_t* drop_b, int64_t n_cap, int64_t* recv,
                                          uint8_t* owned, int64_t* n_recv)
{
    CHECK_ARG(coarse && fine && coarse_lo && coarse_dims && fine_lo && fine_dims && m_b && gamma_b && active_b &&
                  m_s && mb_s && active_s && drop_b && n_recv,
              "NULL argument");
    CHECK_ARG(coarse->dim == fine->dim && (coarse->dim == 2 || coarse->dim == 3), "dim must be 2 or 3 on both");
    auto mk = [](const osmpm_grid_desc* g, const int64_t* lo, const int64_t* nn) {
        HostBox h{};
        h.d = g->dim;
        h.dx = g->dx;
        for (int a = 0; a < 3; ++a) {
            h.o[a] = g->origin[a];
            h.gd[a] = a < g->dim ? g->dims[a] : 1;
            h.lo[a] = a < g->dim ? lo[a] : 0;
            h.nn[a] = a < g->dim ? nn[a] : 1;
        }
        return h;
    };
    std::map<int64_t, char> cand;
    fine_box_receivers(mk(coarse, coarse_lo, coarse_dims), m_b, gamma_b, active_b, mk(fine, fine_lo, fine_dims), nown,
                       m_s, mb_s, active_s, tau_s, drop_b, cand);
    *n_recv = (int64_t)cand.size();
    CHECK_ARG((int64_t)cand.size() <= n_cap || !recv, "receiver capacity n_cap too small");
    if (recv) {
        int64_t q = 0;
        for (auto& kv : cand) {
            recv[q] = kv.first;
            if (owned) owned[q] = (uint8_t)kv.second;
            ++q;
        }
    }
    return OSMPM_OK;
}

osmpm_status osmpm_coupler_create(osmpm_subdomain* coarse, osmpm_subdomain* fine,
                                  const osmpm_schwarz_settings* settings, osmpm_coupler** out)
{
    CHECK_ARG(coarse && fine && settings && out, "NULL argument");
    CHECK_ARG(coarse->dim == fine->dim && coarse->prec == fine->prec, "coupler: subdomains differ in dim / precision");
    CHECK_ARG(coarse->ctx == fine->ctx, "coupler: subdomains belong to different contexts");
    CHECK_ARG(!coarse->decomposed, "coupler: the coarse subdomain must not be decomposed (create it with "
                                   "decompose = 0: it is replicated on every rank)");
    CHECK_ARG(settings->M >= 1, "M must be >= 1");
    CHECK_ARG(settings->k_max >= 1 || settings->parity_fixed_k >= 1, "k_max and parity_fixed_k both < 1: no Schwarz iteration");
    SET_DEVICE(coarse->ctx);
    return coupler_create(coarse, fine, settings, out);
}
void osmpm_coupler_destroy(osmpm_coupler* cpl) { coupler_destroy(cpl); }
osmpm_status osmpm_schwarz_prepare(osmpm_coupler* cpl)
{
    CHECK_ARG(cpl, "coupler is NULL");
    return coupler_prepare(cpl);
}
osmpm_status osmpm_schwarz_substep(osmpm_coupler* cpl, int32_t m, osmpm_solve_stats* stats)
{
    CHECK_ARG(cpl, "coupler is NULL");
    return coupler_substep(cpl, m, stats);
}
osmpm_status osmpm_schwarz_step(osmpm_coupler* cpl, osmpm_schwarz_report* report)
{
    CHECK_ARG(cpl, "coupler is NULL");
    return coupler_step(cpl, report);
}

}  // extern "C"
