// dist.cuh -- a fine subdomain partitioned into x-slabs over the ranks of the context's process
// group (one rank per GPU, NCCL over NVLink / NVSwitch) and, inside a rank, over `local_slabs`
// slabs on the same device.
//
//  * Slab cuts are cell indices along x, chosen at creation from the particles' base-node histogram
//    (balanced particle counts, widths multiples of the tile edge) and fixed afterwards; the first
//    and last slabs are open-ended.  Every rank passes the same full particle view and keeps the
//    particles whose base node lies in its slabs (persistent ids = creation indices).
//  * A particle belongs to the slab containing its base node; its stencil reaches two node planes
//    past the slab, which are the right neighbour's first planes (the ghosts; group.cuh).
//  * After G2P the particles that crossed a cut migrate to the neighbouring slab (device-side
//    classify / reorder / pack, NCCL send-recv between ranks, device copies inside a rank).
#pragma once
#include <memory>

#include "group.cuh"

namespace osmpm {

// 0 stay, 1 left, 2 right by base node x against the slab's cuts; counts[0..2]
template <int D, typename R>
__global__ void k_classify(const R* __restrict__ P, int64_t cap, int64_t n, double o0, double inv_dx, int cut_lo,
                           int cut_hi, uint32_t* __restrict__ keys, int* __restrict__ vals,
                           unsigned long long* __restrict__ counts)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    R f;
    const int b = base_of<R>(P[(PL<D>::X + 0) * cap + p], o0, inv_dx, &f);
    const uint32_t k = (b < cut_lo) ? 1u : (b >= cut_hi ? 2u : 0u);
    keys[p] = k;
    vals[p] = (int)p;
    atomicAdd(&counts[k], 1ull);
}

// movers [i0, i0 + cnt) of the sorted SoA -> contiguous buffer: R fields (nf x cnt), then int
// material and id (2 x cnt), then uint8 boundary flags
template <typename R>
__global__ void k_pack(const R* __restrict__ P, int nf, int64_t cap, int64_t i0, int64_t cnt,
                       const int* __restrict__ mat, const int* __restrict__ pid, const uint8_t* __restrict__ bnd,
                       unsigned char* __restrict__ buf)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    R* bR = reinterpret_cast<R*>(buf);
    int* bI = reinterpret_cast<int*>(buf + ((nf * cnt * sizeof(R) + 15) / 16) * 16);
    uint8_t* bB = reinterpret_cast<uint8_t*>(bI + 2 * cnt);
    for (int f = 0; f < nf; ++f) bR[f * cnt + i] = P[f * cap + i0 + i];
    bI[i] = mat[i0 + i];
    bI[cnt + i] = pid[i0 + i];
    bB[i] = bnd[i0 + i];
}

template <typename R>
__global__ void k_unpack(const unsigned char* __restrict__ buf, int nf, int64_t cap, int64_t i0, int64_t cnt,
                         R* __restrict__ P, int* __restrict__ mat, int* __restrict__ pid, uint8_t* __restrict__ bnd)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const R* bR = reinterpret_cast<const R*>(buf);
    const int* bI = reinterpret_cast<const int*>(buf + ((nf * cnt * sizeof(R) + 15) / 16) * 16);
    const uint8_t* bB = reinterpret_cast<const uint8_t*>(bI + 2 * cnt);
    for (int f = 0; f < nf; ++f) P[f * cap + i0 + i] = bR[f * cnt + i];
    mat[i0 + i] = bI[i];
    pid[i0 + i] = bI[cnt + i];
    bnd[i0 + i] = bB[i];
}

template <typename R>
static size_t pack_bytes(int nf, int64_t cnt)
{
    return ((nf * cnt * sizeof(R) + 15) / 16) * 16 + 2 * cnt * sizeof(int) + cnt + 16;
}

// balanced cuts: nslab - 1 increasing cell indices on the tile-column lattice starting at the lowest
// base node (so every slab width is a multiple of `tile`), each cut the column boundary whose
// prefix particle count is closest to k N / nslab, at least one column per slab
static std::vector<int> balanced_cuts(const std::vector<int>& base_x, int nslab, int tile)
{
    std::vector<int> cuts;
    if (nslab <= 1 || base_x.empty()) return cuts;
    const int bmin = *std::min_element(base_x.begin(), base_x.end());
    const int bmax = *std::max_element(base_x.begin(), base_x.end());
    const int ncol = (bmax - bmin) / tile + 1;  // tile columns
    if (ncol < nslab) return cuts;
    std::vector<int64_t> pre(ncol + 1, 0);
    for (int b : base_x) pre[(b - bmin) / tile + 1]++;
    for (int c = 0; c < ncol; ++c) pre[c + 1] += pre[c];
    const double N = (double)base_x.size();
    int prev = 0;
    for (int k = 1; k < nslab; ++k) {
        const double target = N * k / nslab;
        int best = prev + 1;
        for (int c = prev + 1; c <= ncol - (nslab - k); ++c)
            if (std::fabs(pre[c] - target) < std::fabs(pre[best] - target)) best = c;
        cuts.push_back(bmin + best * tile);
        prev = best;
    }
    return cuts;
}

template <int D, typename R>
struct Dist : public osmpm_subdomain {
    using L = PL<D>;
    std::vector<std::unique_ptr<Sub<D, R>>> own;
    std::vector<Sub<D, R>*> sp;
    GroupBufs gb;
    GroupComm* gc = nullptr;
    int nslab_total = 1, first_slab = 0;
    std::vector<int> cuts;
    double origin[3] = {0, 0, 0}, dx = 1;
    int64_t gdims[3] = {1, 1, 1};
    int64_t n_total = 0;
    double total_mass = 0.0;  // of the whole subdomain (every rank sees the full view)
    DBuf<double> dense_io;          // dense node / creation-order particle staging
    DBuf<unsigned char> mig_recv[2];  // migration payload from the left / right rank
    DBuf<unsigned long long> mig_cnt;
    std::vector<std::unique_ptr<DBuf<unsigned char>>> sendL, sendR;  // per local slab
    unsigned long long* h_cnt = nullptr;

    ~Dist() override
    {
        if (h_cnt) cudaFreeHost(h_cnt);
    }
    cudaStream_t st() const { return ctx->stream; }
    SlabGroup<D, R> group() { return SlabGroup<D, R>{sp.data(), (int)sp.size(), gc, &gb, st(), ctx}; }
    void KC() const { ctx->launches++; }

    osmpm_status create(const osmpm_grid_desc* gd, double dt, const osmpm_particles_view* pv, const osmpm_material* mt,
                        int nm, const double* gravity)
    {
        gc = &ctx->gc;
        OSMPM_TRY(gb.init());
        OSMPM_CU(cudaMallocHost((void**)&h_cnt, 8 * sizeof(unsigned long long)));
        OSMPM_TRY(mig_cnt.need(8));
        for (int a = 0; a < 3; ++a) {
            origin[a] = gd->origin[a];
            gdims[a] = a < D ? gd->dims[a] : 1;
        }
        dx = gd->dx;
        n_total = pv->n;
        const int L_ = std::max(1, gc->local_slabs);
        nslab_total = gc->nranks * L_;
        first_slab = gc->rank * L_;
        // base node x of every particle (all ranks see the same view -> the same cuts)
        std::vector<double> xs((size_t)pv->n * D);
        if (pv->n) {
            if (pv->space == OSMPM_HOST)
                std::memcpy(xs.data(), pv->x, xs.size() * sizeof(double));
            else
                OSMPM_CU(cudaMemcpy(xs.data(), pv->x, xs.size() * sizeof(double), cudaMemcpyDeviceToHost));
        }
        // same arithmetic as the device's base_of (particle precision, then fp64 scaling)
        std::vector<int> bx(pv->n);
        const double inv_dx = 1.0 / dx;
        for (int64_t i = 0; i < pv->n; ++i)
            bx[i] = (int)std::floor(((double)(R)xs[i * D] - origin[0]) * inv_dx - 0.5);
        cuts = balanced_cuts(bx, nslab_total, Tile<D>::T0);
        if ((int)cuts.size() != nslab_total - 1 && nslab_total > 1 && pv->n > 0) {
            set_error("cannot cut %d slabs", nslab_total);
            return OSMPM_E_INVALID_ARG;
        }
        // global activity threshold (R4) from the median particle mass of the whole set
        double med = 0.0;
        if (pv->n > 0) {
            std::vector<double> ms(pv->n);
            if (pv->space == OSMPM_HOST)
                std::memcpy(ms.data(), pv->m, ms.size() * sizeof(double));
            else
                OSMPM_CU(cudaMemcpy(ms.data(), pv->m, ms.size() * sizeof(double), cudaMemcpyDeviceToHost));
            std::sort(ms.begin(), ms.end());
            med = (pv->n % 2) ? ms[pv->n / 2] : 0.5 * (ms[pv->n / 2 - 1] + ms[pv->n / 2]);
            total_mass = 0.0;
            for (double mm : ms) total_mass += mm;
        }
        for (int k = 0; k < L_; ++k) {
            const int gs = first_slab + k;
            const int lo = gs == 0 ? INT32_MIN : cuts[gs - 1];
            const int hi = gs == nslab_total - 1 ? INT32_MAX : cuts[gs];
            std::vector<int64_t> sel;
            for (int64_t i = 0; i < pv->n; ++i)
                if (bx[i] >= lo && bx[i] < hi) sel.push_back(i);
            auto s = std::make_unique<Sub<D, R>>();
            s->ctx = ctx;
            s->dim = D;
            s->prec = prec;
            const int64_t nsel = (int64_t)sel.size();
            OSMPM_TRY(s->create(gd, dt, pv, mt, nm, gravity, sel.data(), nsel, nsel + nsel / 4 + 1024));
            s->cut_lo = lo;
            s->cut_hi = hi;
            s->median_mass = med;
            s->mass_thr = 1e-12 * med;
            sp.push_back(s.get());
            own.push_back(std::move(s));
        }
        // the safe-interior check of every particle
        for (auto* s : sp) {
            int l[3], h[3];
            OSMPM_TRY(s->bounds_local(l, h));
            OSMPM_TRY(s->check_err());
        }
        return migrate();  // no-op unless host and device disagree on a base node
    }

    // ------------------------------------------------------------------------------------------
    osmpm_status set_gravity(const double* g) override
    {
        for (auto* s : sp) OSMPM_TRY(s->set_gravity(g));
        return OSMPM_OK;
    }
    osmpm_status set_dt(double d) override
    {
        for (auto* s : sp) OSMPM_TRY(s->set_dt(d));
        return OSMPM_OK;
    }
    osmpm_status sync() override
    {
        for (auto* s : sp) OSMPM_TRY(s->sync());
        return OSMPM_OK;
    }
    osmpm_status p2g() override { return group_p2g<D, R>(group()); }

    osmpm_status set_dirichlet(int64_t nd, const int64_t* idx, const uint8_t* mask, const double* vel,
                               osmpm_memspace spc) override
    {
        for (auto* s : sp) OSMPM_TRY(s->set_dirichlet(nd, idx, mask, vel, spc));
        return OSMPM_OK;
    }

    // ---- dense node vectors: every slab writes its OWNED nodes, ghosts come from their owner ------
    int64_t dense_nodes() const { return gdims[0] * gdims[1] * gdims[2]; }
    osmpm_status export_field(const std::vector<const double*>& src, int nc, double* dst, osmpm_memspace spc)
    {
        const size_t cnt = (size_t)dense_nodes() * nc;
        double* d = dst;
        if (spc == OSMPM_HOST) {
            OSMPM_TRY(dense_io.need(cnt));
            d = dense_io.p;
        }
        OSMPM_CU(cudaMemsetAsync(d, 0, cnt * sizeof(double), st()));
        for (size_t i = 0; i < sp.size(); ++i) {
            Sub<D, R>* s = sp[i];
            if (!s->have_grid) continue;
            KC();
            k_box_to_dense<D, double><<<nblk_all(s->box.nnodes, 256), 256, 0, st()>>>(s->box, s->nown, nc, src[i], d);
            OSMPM_LAUNCH_CHECK();
        }
        if (spc == OSMPM_HOST) {
            OSMPM_CU(cudaMemcpyAsync(dst, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
        }
        return OSMPM_OK;
    }
    template <typename F>
    osmpm_status export_of(F sel, int nc, double* dst, osmpm_memspace spc)
    {
        std::vector<const double*> src;
        for (auto* s : sp) src.push_back(sel(s));
        return export_field(src, nc, dst, spc);
    }
    osmpm_status import_field(const double* src, int nc, osmpm_memspace spc, DBuf<double> Sub<D, R>::* f)
    {
        const size_t cnt = (size_t)dense_nodes() * nc;
        const double* srcd = src;
        if (spc == OSMPM_HOST) {
            OSMPM_TRY(dense_io.need(cnt));
            OSMPM_CU(cudaMemcpyAsync(dense_io.p, src, cnt * sizeof(double), cudaMemcpyHostToDevice, st()));
            srcd = dense_io.p;
        }
        for (auto* s : sp) OSMPM_TRY(s->import_dense(srcd, nc, (s->*f).p, OSMPM_DEVICE));
        if (spc == OSMPM_HOST) OSMPM_CU(cudaStreamSynchronize(st()));
        return OSMPM_OK;
    }
    osmpm_status need_grid()
    {
        for (auto* s : sp) OSMPM_TRY(s->need_grid());
        return OSMPM_OK;
    }

    osmpm_status read_grid(double* mo, double* po, double* vo, double* fe, double* fs, uint8_t* ao,
                           osmpm_memspace spc) override
    {
        OSMPM_TRY(need_grid());
        if (mo) OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->m.p; }, 1, mo, spc));
        if (po) OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->mom.p; }, D, po, spc));
        if (vo) OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->vn.p; }, D, vo, spc));
        if (fs) OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->fsig.p; }, D, fs, spc));
        if (fe) {
            for (auto* s : sp) {
                const size_t nn = s->box.nnodes;
                OSMPM_TRY(s->tmp.need(nn * D));
                KC();
                k_fext<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, s->m.p, s->grav[0], s->grav[1], s->grav[2], s->tmp.p);
                OSMPM_LAUNCH_CHECK();
            }
            OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->tmp.p; }, D, fe, spc));
        }
        if (ao) {
            const size_t cnt = (size_t)dense_nodes();
            DBuf<uint8_t> tmpa;
            uint8_t* d = ao;
            if (spc == OSMPM_HOST) {
                OSMPM_TRY(tmpa.need(cnt));
                d = tmpa.p;
            }
            OSMPM_CU(cudaMemsetAsync(d, 0, cnt, st()));
            for (auto* s : sp) {
                KC();
                k_box_to_dense<D, uint8_t><<<nblk_all(s->box.nnodes, 256), 256, 0, st()>>>(s->box, s->nown, 1, s->act.p,
                                                                                          d);
                OSMPM_LAUNCH_CHECK();
            }
            if (spc == OSMPM_HOST) {
                OSMPM_CU(cudaMemcpyAsync(ao, d, cnt, cudaMemcpyDeviceToHost, st()));
                OSMPM_CU(cudaStreamSynchronize(st()));
            }
        }
        return OSMPM_OK;
    }

    osmpm_status newton_gradient(const double* uin, double* gout, double* E, osmpm_memspace spc) override
    {
        OSMPM_TRY(need_grid());
        OSMPM_TRY(import_field(uin, D, spc, &Sub<D, R>::u));
        OSMPM_TRY(group_grad<D, R>(group(), false));
        if (gout) OSMPM_TRY(export_of([](Sub<D, R>* s) { return (const double*)s->g.p; }, D, gout, spc));
        if (E) *E = (gb.h_scal[2] > 0) ? INFINITY : gb.h_scal[0] + gb.h_scal[3];
        return OSMPM_OK;
    }
    osmpm_status newton_hvp(const double* din, double* yout, osmpm_memspace spc) override
    {
        OSMPM_TRY(need_grid());
        for (auto* s : sp)
            if (!s->have_lin) {
                set_error("newton_hvp needs a prior newton_gradient (linearisation point)");
                return OSMPM_E_STATE;
            }
        OSMPM_TRY(import_field(din, D, spc, &Sub<D, R>::p));
        OSMPM_TRY(group_hvp<D, R>(group()));
        return export_of([](Sub<D, R>* s) { return (const double*)s->y.p; }, D, yout, spc);
    }
    osmpm_status newton_diag(double* dout, osmpm_memspace spc) override
    {
        OSMPM_TRY(need_grid());
        for (auto* s : sp)
            if (!s->have_lin) {
                set_error("newton_diag needs a prior newton_gradient");
                return OSMPM_E_STATE;
            }
        return export_of([](Sub<D, R>* s) { return (const double*)s->dg.p; }, D, dout, spc);
    }
    osmpm_status implicit_solve(const osmpm_newton_settings* s, osmpm_solve_stats* stats) override
    {
        OSMPM_TRY(need_grid());
        return group_solve<D, R>(group(), s, stats);
    }
    osmpm_status read_grid_velocity(double* v, osmpm_memspace spc) override
    {
        bool last = true;
        for (auto* s : sp) last = last && s->have_vlast;
        if (!last) {
            OSMPM_TRY(need_grid());
            for (auto* s : sp)
                if (!s->have_vnew) {
                    set_error("no solved grid velocity");
                    return OSMPM_E_STATE;
                }
        }
        return export_of([](Sub<D, R>* s) { return (const double*)s->vnew.p; }, D, v, spc);
    }
    osmpm_status set_grid_velocity(const double* v, osmpm_memspace spc) override
    {
        OSMPM_TRY(need_grid());
        OSMPM_TRY(import_field(v, D, spc, &Sub<D, R>::vnew));
        for (auto* s : sp) s->have_vnew = true;
        return OSMPM_OK;
    }

    // ---- a11: checkpoint / restore every slab (each slab keeps its own count) ---------------------
    osmpm_status checkpoint() override
    {
        for (auto* s : sp) OSMPM_TRY(s->checkpoint());
        return OSMPM_OK;
    }
    osmpm_status restore() override
    {
        for (auto* s : sp) OSMPM_TRY(s->restore());
        return OSMPM_OK;
    }

    // ---- a8: G2P on every slab, then migration across the cuts ---------------------------------
    osmpm_status g2p() override
    {
        for (auto* s : sp) OSMPM_TRY(s->g2p());
        return migrate();
    }

    osmpm_status migrate()
    {
        const int ns = (int)sp.size();
        if (nslab_total == 1) return OSMPM_OK;
        std::vector<int64_t> nstay(ns), nl(ns), nr(ns);
        // classify + reorder [stay | left | right]
        for (int i = 0; i < ns; ++i) {
            Sub<D, R>* s = sp[i];
            OSMPM_TRY(s->check_err());
            OSMPM_CU(cudaMemsetAsync(mig_cnt.p, 0, 3 * sizeof(unsigned long long), st()));
            if (s->n > 0) {
                OSMPM_TRY(s->keys.need(s->cap));
                OSMPM_TRY(s->keys2.need(s->cap));
                OSMPM_TRY(s->vals.need(s->cap));
                OSMPM_TRY(s->vals2.need(s->cap));
                KC();
                k_classify<D, R><<<nblk_all(s->n, 256), 256, 0, st()>>>(s->P.p, s->cap, s->n, origin[0], 1.0 / dx,
                                                                      s->cut_lo, s->cut_hi, s->keys.p, s->vals.p,
                                                                      mig_cnt.p);
                OSMPM_LAUNCH_CHECK();
            }
            OSMPM_CU(cudaMemcpyAsync(h_cnt, mig_cnt.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            nstay[i] = (int64_t)h_cnt[0];
            nl[i] = (int64_t)h_cnt[1];
            nr[i] = (int64_t)h_cnt[2];
            if (nl[i] + nr[i] > 0) {
                OSMPM_TRY(s->rs_hist.need(radix_hist_words(s->n)));
                // 2-bit keys stay / left / right: one stable radix pass (radix_sort.cuh)
                if (!radix_sort_pairs(s->keys.p, s->vals.p, s->keys2.p, s->vals2.p, s->n, 2, s->rs_hist.p, st(),
                                      ctx->launches)) {
                    std::swap(s->keys.p, s->keys2.p);
                    std::swap(s->keys.cap, s->keys2.cap);
                    std::swap(s->vals.p, s->vals2.p);
                    std::swap(s->vals.cap, s->vals2.cap);
                }
                OSMPM_LAUNCH_CHECK();
                KC();
                k_permute<R><<<nblk_all(s->n, 256), 256, 0, st()>>>(s->P.p, s->P2.p, L::NF, s->cap, s->n, s->vals2.p,
                                                                    s->mat.p, s->mat2.p, s->bnd.p, s->bnd2.p, s->pid.p,
                                                                    s->pid2.p);
                OSMPM_LAUNCH_CHECK();
                std::swap(s->P.p, s->P2.p);
                std::swap(s->P.cap, s->P2.cap);
                std::swap(s->mat.p, s->mat2.p);
                std::swap(s->mat.cap, s->mat2.cap);
                std::swap(s->bnd.p, s->bnd2.p);
                std::swap(s->bnd.cap, s->bnd2.cap);
                std::swap(s->pid.p, s->pid2.p);
                std::swap(s->pid.cap, s->pid2.cap);
            }
        }
        // pack every slab's movers (per direction) into its send buffers (grow-only members)
        while ((int)sendL.size() < ns) {
            sendL.push_back(std::make_unique<DBuf<unsigned char>>());
            sendR.push_back(std::make_unique<DBuf<unsigned char>>());
        }
        for (int i = 0; i < ns; ++i) {
            Sub<D, R>* s = sp[i];
            const int64_t c2[2] = {nl[i], nr[i]};
            const int64_t o2[2] = {nstay[i], nstay[i] + nl[i]};
            DBuf<unsigned char>* b2[2] = {sendL[i].get(), sendR[i].get()};
            for (int d = 0; d < 2; ++d) {
                if (c2[d] == 0) continue;
                OSMPM_TRY(b2[d]->need(pack_bytes<R>(L::NF, c2[d])));
                KC();
                k_pack<R><<<nblk_all(c2[d], 256), 256, 0, st()>>>(s->P.p, L::NF, s->cap, o2[d], c2[d], s->mat.p,
                                                                  s->pid.p, s->bnd.p, b2[d]->p);
                OSMPM_LAUNCH_CHECK();
            }
            s->n = nstay[i];
        }
        // append helper
        auto append = [&](Sub<D, R>* s, const unsigned char* buf, int64_t cnt) -> osmpm_status {
            if (cnt == 0) return OSMPM_OK;
            if (s->n + cnt > s->cap - 4) {
                set_error("slab capacity %lld exceeded by migration (%lld + %lld particles)", (long long)s->cap,
                          (long long)s->n, (long long)cnt);
                return OSMPM_E_OOM;
            }
            KC();
            k_unpack<R><<<nblk_all(cnt, 256), 256, 0, st()>>>(buf, L::NF, s->cap, s->n, cnt, s->P.p, s->mat.p, s->pid.p,
                                                              s->bnd.p);
            OSMPM_LAUNCH_CHECK();
            s->n += cnt;
            return OSMPM_OK;
        };
        // inside the rank
        for (int i = 0; i < ns; ++i) {
            if (i > 0) OSMPM_TRY(append(sp[i - 1], sendL[i]->p, nl[i]));
            if (i + 1 < ns) OSMPM_TRY(append(sp[i + 1], sendR[i]->p, nr[i]));
        }
        // across ranks: counts, then payloads
        if (gc->multi()) {
            const int r = gc->rank;
            int64_t* hc = reinterpret_cast<int64_t*>(h_cnt);
            int64_t* dc = reinterpret_cast<int64_t*>(mig_cnt.p);
            hc[0] = nl[0];       // to the left rank
            hc[1] = nr[ns - 1];  // to the right rank
            hc[2] = hc[3] = 0;
            OSMPM_CU(cudaMemcpyAsync(dc, hc, 4 * sizeof(int64_t), cudaMemcpyHostToDevice, st()));
            OSMPM_NCCL(ncclGroupStart());
            if (r > 0) {
                OSMPM_NCCL(ncclSend(dc + 0, 1, ncclInt64, r - 1, gc->comm, st()));
                OSMPM_NCCL(ncclRecv(dc + 2, 1, ncclInt64, r - 1, gc->comm, st()));
            }
            if (r + 1 < gc->nranks) {
                OSMPM_NCCL(ncclSend(dc + 1, 1, ncclInt64, r + 1, gc->comm, st()));
                OSMPM_NCCL(ncclRecv(dc + 3, 1, ncclInt64, r + 1, gc->comm, st()));
            }
            OSMPM_NCCL(ncclGroupEnd());
            OSMPM_CU(cudaMemcpyAsync(hc, dc, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            const int64_t from_left = hc[2], from_right = hc[3];
            if (r > 0 && from_left) OSMPM_TRY(mig_recv[0].need(pack_bytes<R>(L::NF, from_left)));
            if (r + 1 < gc->nranks && from_right) OSMPM_TRY(mig_recv[1].need(pack_bytes<R>(L::NF, from_right)));
            OSMPM_NCCL(ncclGroupStart());
            if (r > 0) {
                if (nl[0]) OSMPM_NCCL(ncclSend(sendL[0]->p, pack_bytes<R>(L::NF, nl[0]), ncclUint8, r - 1, gc->comm, st()));
                if (from_left)
                    OSMPM_NCCL(ncclRecv(mig_recv[0].p, pack_bytes<R>(L::NF, from_left), ncclUint8, r - 1, gc->comm, st()));
            }
            if (r + 1 < gc->nranks) {
                if (nr[ns - 1])
                    OSMPM_NCCL(ncclSend(sendR[ns - 1]->p, pack_bytes<R>(L::NF, nr[ns - 1]), ncclUint8, r + 1, gc->comm,
                                        st()));
                if (from_right)
                    OSMPM_NCCL(
                        ncclRecv(mig_recv[1].p, pack_bytes<R>(L::NF, from_right), ncclUint8, r + 1, gc->comm, st()));
            }
            OSMPM_NCCL(ncclGroupEnd());
            if (r > 0) OSMPM_TRY(append(sp[0], mig_recv[0].p, from_left));
            if (r + 1 < gc->nranks) OSMPM_TRY(append(sp[ns - 1], mig_recv[1].p, from_right));
        }
        return OSMPM_OK;
    }

    // ---- particle I/O in creation order: each rank writes its own particles ----------------------
    osmpm_status read_particles(double* x, double* v, double* F, double* B, osmpm_memspace spc) override
    {
        struct Fld { double* dst; int off, nc; };
        const Fld flds[] = {{x, L::X, D}, {v, L::V, D}, {F, L::F, D * D}, {B, L::B, D * D}};
        for (const Fld& fl : flds) {
            if (!fl.dst || n_total == 0) continue;
            const size_t cnt = (size_t)n_total * fl.nc;
            double* d = fl.dst;
            if (spc == OSMPM_HOST) {
                OSMPM_TRY(dense_io.need(cnt));
                d = dense_io.p;
                OSMPM_CU(cudaMemsetAsync(d, 0, cnt * sizeof(double), st()));
            }
            for (auto* s : sp)
                for (int c = 0; c < fl.nc; ++c) {
                    if (s->n == 0) continue;
                    KC();
                    k_unsort_field<R><<<nblk_all(s->n, 256), 256, 0, st()>>>(s->P.p + (size_t)(fl.off + c) * s->cap, s->n,
                                                                           s->pid.p, fl.nc, c, d);
                }
            OSMPM_LAUNCH_CHECK();
            if (spc == OSMPM_HOST) {
                OSMPM_CU(cudaMemcpyAsync(fl.dst, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, st()));
                OSMPM_CU(cudaStreamSynchronize(st()));
            }
        }
        return OSMPM_OK;
    }
    osmpm_status set_particles(const double* x, const double* v, const double* F, const double* B,
                               osmpm_memspace spc) override
    {
        struct Fld { const double* src; int off, nc; };
        const Fld flds[] = {{x, L::X, D}, {v, L::V, D}, {F, L::F, D * D}, {B, L::B, D * D}};
        for (const Fld& fl : flds) {
            if (!fl.src || n_total == 0) continue;
            const size_t cnt = (size_t)n_total * fl.nc;
            const double* srcd = fl.src;
            if (spc == OSMPM_HOST) {
                OSMPM_TRY(dense_io.need(cnt));
                OSMPM_CU(cudaMemcpyAsync(dense_io.p, fl.src, cnt * sizeof(double), cudaMemcpyHostToDevice, st()));
                srcd = dense_io.p;
            }
            for (auto* s : sp)
                for (int c = 0; c < fl.nc; ++c) {
                    if (s->n == 0) continue;
                    KC();
                    k_sort_field<R><<<nblk_all(s->n, 256), 256, 0, st()>>>(srcd, s->n, s->pid.p, fl.nc, c,
                                                                         s->P.p + (size_t)(fl.off + c) * s->cap);
                }
            OSMPM_LAUNCH_CHECK();
            if (spc == OSMPM_HOST) OSMPM_CU(cudaStreamSynchronize(st()));
        }
        for (auto* s : sp) s->have_grid = s->have_lin = s->have_vnew = false;
        return migrate();  // new positions may lie in other slabs
    }

    osmpm_status info(int64_t* np, int64_t* lo, int64_t* dims) override
    {
        int64_t nl = 0;
        for (auto* s : sp) nl += s->n;
        if (np) *np = nl;
        for (int a = 0; a < 3; ++a) {
            const BoxDev& b0 = sp.front()->box;
            const BoxDev& b1 = sp.back()->box;
            if (lo) lo[a] = b0.lo[a];
            if (dims) dims[a] = (a == 0) ? (b1.lo[0] + b1.nn[0] - b0.lo[0]) : b0.nn[a];
        }
        return OSMPM_OK;
    }
};

}  // namespace osmpm
