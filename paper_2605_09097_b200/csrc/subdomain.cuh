// subdomain.cuh -- one MPM subdomain on one GPU (§3.1: its own grid dx, time step dt and
// particle set), templated on dimension D and particle precision R.
#pragma once
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <vector>

#include "kernels.cuh"
#include "runtime.h"

namespace osmpm {

template <typename T>
static osmpm_status ensure(T*& p, size_t& cap, size_t n)
{
    if (n <= cap && p) return OSMPM_OK;
    if (p) cudaFree(p);
    p = nullptr;
    size_t want = std::max<size_t>(n + n / 8, 64);
    cudaError_t e = cudaMalloc((void**)&p, want * sizeof(T));
    if (e != cudaSuccess) {
        cap = 0;
        set_error("cudaMalloc(%zu bytes) failed: %s", want * sizeof(T), cudaGetErrorString(e));
        return OSMPM_E_OOM;
    }
    cap = want;
    return OSMPM_OK;
}

template <typename T> struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    osmpm_status need(size_t n) { return ensure(p, cap, n); }
    ~DBuf()
    {
        if (p) cudaFree(p);
    }
};

static inline int nblk(int64_t n, int bs, int maxb = 148 * 8)
{
    int64_t b = (n + bs - 1) / bs;
    if (b < 1) b = 1;
    return (int)std::min<int64_t>(b, maxb);
}
static inline int nblk_all(int64_t n, int bs)
{
    int64_t b = (n + bs - 1) / bs;
    return (int)std::max<int64_t>(b, 1);
}

// A Dirichlet list in global dense-box node indices (user constraints, or Schwarz receivers)
struct DirList {
    DBuf<int64_t> idx;
    DBuf<uint8_t> mask;
    DBuf<double> val;
    int64_t n = 0;
};

template <int D, typename R>
struct Sub : public osmpm_subdomain {
    using L = PL<D>;
    using C = CL<D>;
    using T = Tile<D>;

    // ---- configuration ----------------------------------------------------------------------
    double origin[3] = {0, 0, 0}, dx = 1, dt = 1, grav[3] = {0, 0, 0};
    int64_t gdims[3] = {1, 1, 1};
    MatTable mats{};
    double mass_thr = 0;  // 1e-12 * median m_p (R4)
    int64_t n = 0, cap = 0;

    // ---- particles (sorted) -----------------------------------------------------------------
    DBuf<R> P, P2, cache, Pck;
    DBuf<int> mat, mat2, pid, pid2, matck, pidck;
    DBuf<uint8_t> bnd, bnd2, bndck;
    bool have_ck = false;
    DBuf<uint32_t> keys, keys2;
    DBuf<int> vals, vals2;
    DBuf<unsigned char> cub_tmp;

    // ---- node box ---------------------------------------------------------------------------
    BoxDev box{};
    bool have_grid = false, have_lin = false, have_vnew = false;
    DBuf<int> cell_start;
    DBuf<double> m, mom, vn, fsig, mb, dval, u, g, dg, xs, r, z, p, y, ut, vnew, tmp;
    DBuf<uint8_t> act, dmask, fmask;
    DirList dir_user, dir_cpl;
    DBuf<double> stage_io;  // persistent host-I/O staging buffer

    // ---- reductions / scalars ---------------------------------------------------------------
    DBuf<double> partA, partB, scal;
    DBuf<CGScalars> cgs;
    DBuf<ErrLatch> err;
    DBuf<int> bounds;
    double* h_scal = nullptr;  // pinned
    CGScalars* h_cgs = nullptr;
    int* h_bounds = nullptr;

    ~Sub() override
    {
        if (h_scal) cudaFreeHost(h_scal);
        if (h_cgs) cudaFreeHost(h_cgs);
        if (h_bounds) cudaFreeHost(h_bounds);
    }

    cudaStream_t st() const { return ctx->stream; }
    void KC() const { ctx->launches++; }

    // =========================================================================================
    // creation
    // =========================================================================================
    osmpm_status create(const osmpm_grid_desc* gd, double dt_, const osmpm_particles_view* pv,
                        const osmpm_material* mt, int nm, const double* gravity)
    {
        for (int a = 0; a < 3; ++a) {
            origin[a] = gd->origin[a];
            gdims[a] = a < D ? gd->dims[a] : 1;
            grav[a] = gravity ? gravity[a] : 0.0;
        }
        dx = gd->dx;
        dt = dt_;
        if (nm < 1 || nm > MAX_MATS) {
            set_error("n_mats = %d outside [1, %d]", nm, MAX_MATS);
            return OSMPM_E_INVALID_ARG;
        }
        mats.n = nm;
        for (int k = 0; k < nm; ++k) {
            mats.mu[k] = mt[k].E / (2.0 * (1.0 + mt[k].nu));
            mats.lam[k] = mt[k].E * mt[k].nu / ((1.0 + mt[k].nu) * (1.0 - 2.0 * mt[k].nu));
        }
        n = pv->n;
        // field stride: a multiple of 4 (16-B aligned fields for the TMA bulk copies) with >= 4
        // elements of slack (bulk copies round their length up to 16 B)
        cap = ((n + 4 + 3) / 4) * 4;
        OSMPM_CU(cudaMallocHost((void**)&h_scal, 64 * sizeof(double)));
        OSMPM_CU(cudaMallocHost((void**)&h_cgs, sizeof(CGScalars)));
        OSMPM_CU(cudaMallocHost((void**)&h_bounds, 8 * sizeof(int)));
        OSMPM_TRY(P.need(L::NF * cap));
        OSMPM_TRY(P2.need(L::NF * cap));
        OSMPM_TRY(cache.need(C::NF * cap));
        OSMPM_TRY(mat.need(cap));
        OSMPM_TRY(mat2.need(cap));
        OSMPM_TRY(pid.need(cap));
        OSMPM_TRY(pid2.need(cap));
        OSMPM_TRY(bnd.need(cap));
        OSMPM_TRY(bnd2.need(cap));
        OSMPM_TRY(err.need(1));
        OSMPM_TRY(bounds.need(8));
        OSMPM_TRY(scal.need(64));
        OSMPM_TRY(cgs.need(1));
        OSMPM_CU(cudaMemsetAsync(err.p, 0, sizeof(ErrLatch), st()));
        // host staging in creation order -> field-major SoA (the initial order is creation order)
        std::vector<R> h((size_t)L::NF * cap);
        std::vector<int> hm(cap, 0), hp(cap);
        std::vector<uint8_t> hb(cap, 0);
        std::vector<double> tmpd;
        auto host_view = [&](const double* src, size_t cnt) -> const double* {
            if (!src) return nullptr;
            if (pv->space == OSMPM_HOST) return src;
            tmpd.resize(cnt);
            cudaMemcpy(tmpd.data(), src, cnt * sizeof(double), cudaMemcpyDeviceToHost);
            return tmpd.data();
        };
        struct Fld { const double* src; int off, nc; };
        const Fld flds[] = {{pv->x, L::X, D}, {pv->v, L::V, D}, {pv->F, L::F, D * D},
                            {pv->B, L::B, D * D}, {pv->m, L::M, 1}, {pv->V0, L::VOL, 1}};
        for (const Fld& fl : flds) {
            const double* s = host_view(fl.src, (size_t)n * fl.nc);
            for (int c = 0; c < fl.nc; ++c)
                for (int64_t i = 0; i < n; ++i) {
                    double v = s ? s[i * fl.nc + c] : ((fl.off == L::F || fl.off == L::B) ? 0.0 : 0.0);
                    if (!s && fl.off == L::F && (c % (D + 1)) == 0) v = 1.0;
                    h[(size_t)(fl.off + c) * cap + i] = (R)v;
                }
        }
        if (pv->material) {
            if (pv->space == OSMPM_HOST)
                std::memcpy(hm.data(), pv->material, n * sizeof(int));
            else
                cudaMemcpy(hm.data(), pv->material, n * sizeof(int), cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < n; ++i)
                if (hm[i] < 0 || hm[i] >= nm) {
                    set_error("particle %lld: material %d outside [0, %d)", (long long)i, hm[i], nm);
                    return OSMPM_E_INVALID_ARG;
                }
        }
        if (pv->is_boundary) {
            if (pv->space == OSMPM_HOST)
                std::memcpy(hb.data(), pv->is_boundary, n);
            else
                cudaMemcpy(hb.data(), pv->is_boundary, n, cudaMemcpyDeviceToHost);
        }
        for (int64_t i = 0; i < n; ++i) hp[i] = (int)i;
        // activity threshold 1e-12 * median particle mass (R4)
        if (n > 0) {
            std::vector<double> ms(n);
            for (int64_t i = 0; i < n; ++i) ms[i] = (double)h[(size_t)L::M * cap + i];
            std::sort(ms.begin(), ms.end());
            double med = (n % 2) ? ms[n / 2] : 0.5 * (ms[n / 2 - 1] + ms[n / 2]);
            mass_thr = 1e-12 * med;
            median_mass = med;
            total_mass = 0.0;
            for (double mm : ms) total_mass += mm;
        }
        OSMPM_CU(cudaMemcpy(P.p, h.data(), h.size() * sizeof(R), cudaMemcpyHostToDevice));
        OSMPM_CU(cudaMemcpy(mat.p, hm.data(), cap * sizeof(int), cudaMemcpyHostToDevice));
        OSMPM_CU(cudaMemcpy(pid.p, hp.data(), cap * sizeof(int), cudaMemcpyHostToDevice));
        OSMPM_CU(cudaMemcpy(bnd.p, hb.data(), cap, cudaMemcpyHostToDevice));
        // validate the safe interior right away
        OSMPM_TRY(compute_box());
        return check_err();
    }
    double median_mass = 0, total_mass = 0;

    osmpm_status set_gravity(const double* gv) override
    {
        for (int a = 0; a < 3; ++a) grav[a] = gv[a];
        return OSMPM_OK;
    }
    osmpm_status set_dt(double d) override
    {
        if (!(d > 0)) {
            set_error("dt must be > 0");
            return OSMPM_E_INVALID_ARG;
        }
        dt = d;
        return OSMPM_OK;
    }

    // =========================================================================================
    // errors
    // =========================================================================================
    osmpm_status check_err()
    {
        ErrLatch h{};
        OSMPM_CU(cudaMemcpyAsync(&h, err.p, sizeof(ErrLatch), cudaMemcpyDeviceToHost, st()));
        OSMPM_CU(cudaStreamSynchronize(st()));
        if (h.code) {
            OSMPM_CU(cudaMemsetAsync(err.p, 0, sizeof(ErrLatch), st()));
            if (h.code == OSMPM_E_OUT_OF_DOMAIN)
                set_error("particle %lld left the safe interior of the node box", h.index);
            else if (h.code == OSMPM_E_INVERTED_F)
                set_error("particle %lld: det F <= 0 after G2P", h.index);
            else
                set_error("device error %d (particle %lld)", h.code, h.index);
            return (osmpm_status)h.code;
        }
        return OSMPM_OK;
    }
    osmpm_status sync() override
    {
        OSMPM_CU(cudaStreamSynchronize(st()));
        return check_err();
    }

    // =========================================================================================
    // a1: box + sort
    // =========================================================================================
    void fill_box_common(BoxDev& b) const
    {
        for (int a = 0; a < 3; ++a) {
            b.o[a] = origin[a];
            b.gdims[a] = (int)gdims[a];
        }
        b.dx = dx;
        b.inv_dx = 1.0 / dx;
    }

    osmpm_status compute_box()
    {
        BoxDev b{};
        fill_box_common(b);
        int init[8] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN, 0, 0};
        OSMPM_CU(cudaMemcpyAsync(bounds.p, init, sizeof(init), cudaMemcpyHostToDevice, st()));
        if (n > 0) {
            KC(); k_bounds<D, R><<<nblk(n, 256), 256, 0, st()>>>(P.p, cap, n, b, bounds.p, pid.p, err.p);
            OSMPM_LAUNCH_CHECK();
        }
        OSMPM_CU(cudaMemcpyAsync(h_bounds, bounds.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, st()));
        OSMPM_CU(cudaStreamSynchronize(st()));
        const int tt[3] = {T::T0, T::T1, T::T2};
        int64_t ncells = 1, nnodes = 1;
        int ntiles = 1;
        for (int a = 0; a < 3; ++a) {
            if (a < D && n > 0) {
                int lo = h_bounds[a], hi = h_bounds[3 + a];
                int c = hi - lo + 1;
                c = ((c + tt[a] - 1) / tt[a]) * tt[a];
                b.lo[a] = lo;
                b.nc[a] = c;
                b.nn[a] = c + 2;
                b.nt[a] = c / tt[a];
            } else if (a < D) {
                b.lo[a] = 0;
                b.nc[a] = tt[a];
                b.nn[a] = tt[a] + 2;
                b.nt[a] = 1;
            } else {
                b.lo[a] = 0;
                b.nc[a] = 1;
                b.nn[a] = 1;
                b.nt[a] = 1;
            }
            ncells *= b.nc[a];
            nnodes *= b.nn[a];
            ntiles *= b.nt[a];
        }
        b.ncells = ncells;
        b.nnodes = nnodes;
        b.ntiles = ntiles;
        box = b;
        return OSMPM_OK;
    }

    osmpm_status sort_particles()
    {
        if (n == 0) return OSMPM_OK;
        OSMPM_TRY(keys.need(cap));
        OSMPM_TRY(keys2.need(cap));
        OSMPM_TRY(vals.need(cap));
        OSMPM_TRY(vals2.need(cap));
        OSMPM_TRY(cell_start.need(box.ncells + 1));
        auto& pf = ctx->prof;
        if (pf.on) pf.begin("sort", st());
        KC(); k_keys<D, R><<<nblk_all(n, 256), 256, 0, st()>>>(P.p, cap, n, box, keys.p, vals.p);
        OSMPM_LAUNCH_CHECK();
        int nbits = 1;
        while ((int64_t(1) << nbits) < box.ncells) ++nbits;
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p, (int)n, 0, nbits, st());
        OSMPM_TRY(cub_tmp.need(bytes));
        OSMPM_CU(cub::DeviceRadixSort::SortPairs(cub_tmp.p, bytes, keys.p, keys2.p, vals.p, vals2.p, (int)n, 0,
                                                 nbits, st()));
        KC(); k_permute<R><<<nblk_all(n, 256), 256, 0, st()>>>(P.p, P2.p, L::NF, cap, n, vals2.p, mat.p, mat2.p, bnd.p,
                                                         bnd2.p, pid.p, pid2.p);
        OSMPM_LAUNCH_CHECK();
        std::swap(P.p, P2.p);
        std::swap(P.cap, P2.cap);
        std::swap(mat.p, mat2.p);
        std::swap(mat.cap, mat2.cap);
        std::swap(bnd.p, bnd2.p);
        std::swap(bnd.cap, bnd2.cap);
        std::swap(pid.p, pid2.p);
        std::swap(pid.cap, pid2.cap);
        KC(); k_cell_start<<<nblk_all(n + 1, 256), 256, 0, st()>>>(keys2.p, n, box.ncells, cell_start.p);
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("sort", st());
        return OSMPM_OK;
    }

    osmpm_status alloc_nodes()
    {
        const size_t nn = box.nnodes, nd = nn * D;
        for (DBuf<double>* b : {&m, &mb})
            OSMPM_TRY(b->need(nn));
        for (DBuf<double>* b : {&mom, &vn, &fsig, &dval, &u, &g, &dg, &xs, &r, &z, &p, &y, &ut, &vnew})
            OSMPM_TRY(b->need(nd));
        OSMPM_TRY(act.need(nn));
        OSMPM_TRY(dmask.need(nn));
        OSMPM_TRY(fmask.need(nd));
        OSMPM_TRY(partA.need((size_t)std::max<int64_t>(box.ntiles, 148 * 8) * 4));
        OSMPM_TRY(partB.need((size_t)148 * 8 * 4));
        return OSMPM_OK;
    }

    // =========================================================================================
    // a2: P2G
    // =========================================================================================
    osmpm_status p2g() override
    {
        OSMPM_TRY(compute_box());
        OSMPM_TRY(check_err());
        OSMPM_TRY(sort_particles());
        OSMPM_TRY(alloc_nodes());
        const size_t nn = box.nnodes;
        OSMPM_CU(cudaMemsetAsync(m.p, 0, nn * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(mom.p, 0, nn * D * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(fsig.p, 0, nn * D * sizeof(double), st()));
        auto& pf = ctx->prof;
        if (pf.on) pf.begin("p2g", st());
        if (n > 0) {
            KC(); k_p2g<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, mat.p, box, mats, m.p, mom.p, fsig.p);
            OSMPM_LAUNCH_CHECK();
        }
        KC(); k_p2g_nodes<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, m.p, mom.p, vn.p, act.p, mass_thr);
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("p2g", st());
        have_grid = true;
        have_lin = false;
        have_vnew = false;
        return OSMPM_OK;
    }

    osmpm_status boundary_mass()
    {
        OSMPM_CU(cudaMemsetAsync(mb.p, 0, box.nnodes * sizeof(double), st()));
        if (n > 0) {
            KC(); k_bmass<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, bnd.p, box, mb.p);
            OSMPM_LAUNCH_CHECK();
        }
        return OSMPM_OK;
    }

    // =========================================================================================
    // dense <-> box helpers
    // =========================================================================================
    int64_t dense_nodes() const { return gdims[0] * gdims[1] * gdims[2]; }

    template <typename Tv>
    osmpm_status export_dense(const Tv* src, int nc, Tv* dst, osmpm_memspace sp)
    {
        const size_t cnt = (size_t)dense_nodes() * nc;
        Tv* dptr = dst;
        DBuf<Tv> local;
        DBuf<Tv>* stage = &local;
        if constexpr (std::is_same<Tv, double>::value) stage = &stage_io;
        if (sp == OSMPM_HOST) {
            OSMPM_TRY(stage->need(cnt));
            dptr = stage->p;
        }
        OSMPM_CU(cudaMemsetAsync(dptr, 0, cnt * sizeof(Tv), st()));
        if (have_grid) {
            KC(); k_box_to_dense<D, Tv><<<nblk_all(box.nnodes, 256), 256, 0, st()>>>(box, nc, src, dptr);
            OSMPM_LAUNCH_CHECK();
        }
        if (sp == OSMPM_HOST) {
            OSMPM_CU(cudaMemcpyAsync(dst, dptr, cnt * sizeof(Tv), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
        }
        return OSMPM_OK;
    }

    osmpm_status import_dense(const double* src, int nc, double* dst, osmpm_memspace sp)
    {
        const size_t cnt = (size_t)dense_nodes() * nc;
        const double* sptr = src;
        DBuf<double>& stage = stage_io;
        if (sp == OSMPM_HOST) {
            OSMPM_TRY(stage.need(cnt));
            OSMPM_CU(cudaMemcpyAsync(stage.p, src, cnt * sizeof(double), cudaMemcpyHostToDevice, st()));
            sptr = stage.p;
        }
        KC(); k_dense_to_box<D, double><<<nblk_all(box.nnodes, 256), 256, 0, st()>>>(box, nc, sptr, dst);
        OSMPM_LAUNCH_CHECK();
        if (sp == OSMPM_HOST) OSMPM_CU(cudaStreamSynchronize(st()));
        return OSMPM_OK;
    }

    osmpm_status need_grid()
    {
        if (!have_grid) {
            set_error("no grid: call osmpm_p2g first");
            return OSMPM_E_STATE;
        }
        return OSMPM_OK;
    }

    osmpm_status read_grid(double* mo, double* po, double* vo, double* fe, double* fs, uint8_t* ao,
                           osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        const size_t nn = box.nnodes;
        if (mo) OSMPM_TRY(export_dense<double>(m.p, 1, mo, sp));
        if (po) OSMPM_TRY(export_dense<double>(mom.p, D, po, sp));
        if (vo) OSMPM_TRY(export_dense<double>(vn.p, D, vo, sp));
        if (fs) OSMPM_TRY(export_dense<double>(fsig.p, D, fs, sp));
        if (ao) OSMPM_TRY(export_dense<uint8_t>(act.p, 1, ao, sp));
        if (fe) {
            // f_ext = m g (PAPER.md:178 with partition of unity)
            OSMPM_TRY(tmp.need(nn * D));
            KC(); k_fext<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, m.p, grav[0], grav[1], grav[2], tmp.p);
            OSMPM_LAUNCH_CHECK();
            OSMPM_TRY(export_dense<double>(tmp.p, D, fe, sp));
        }
        return OSMPM_OK;
    }



    // =========================================================================================
    // a4: gradient + energy at u (box vector) -> g (raw), dg (raw), scalars
    // scal[0..2] particle {E, |E|, inverted}; scal[3..5] node {E, |E|, |g_free|^2}
    // =========================================================================================
    size_t grad_smem() const { return grad_smem_bytes<D>(); }
    size_t hvp_smem() const { return hvp_smem_bytes<D, R>(); }

    osmpm_status grad_eval(const double* uu, bool need_fmask)
    {
        const size_t nn = box.nnodes;
        OSMPM_TRY(cache.need(C::NF * cap));
        OSMPM_CU(cudaMemsetAsync(g.p, 0, nn * D * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(dg.p, 0, nn * D * sizeof(double), st()));
        if (!need_fmask) OSMPM_CU(cudaMemsetAsync(fmask.p, 1, nn * D, st()));
        auto& pf = ctx->prof;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_grad<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad_smem());
            cudaFuncSetAttribute(k_hvp<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hvp_smem());
            attr = true;
        }
        if (pf.on) pf.begin("grad", st());
        KC(); k_grad<D, R><<<box.ntiles, T::NT, grad_smem(), st()>>>(P.p, cache.p, cap, mat.p, cell_start.p, box, mats,
                                                               uu, g.p, dg.p, partA.p);
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("grad", st());
        const int nbn = nblk(nn, 256);
        KC(); k_grad_nodes<D><<<nbn, 256, 0, st()>>>(nn, m.p, vn.p, uu, fmask.p, dt, grav[0], grav[1], grav[2], g.p, dg.p,
                                                partB.p);
        OSMPM_LAUNCH_CHECK();
        // scal[0..2] particles {E, E_abs, inverted}; scal[3..6] nodes {E, E_abs, |g_free|^2, f_scale^2}
        KC(); k_final_sum<3><<<1, 1024, 0, st()>>>(partA.p, box.ntiles, scal.p);
        KC(); k_final_sum<4><<<1, 1024, 0, st()>>>(partB.p, nbn, scal.p + 3);
        OSMPM_LAUNCH_CHECK();
        have_lin = true;
        return OSMPM_OK;
    }

    osmpm_status read_scal(int cnt)
    {
        OSMPM_CU(cudaMemcpyAsync(h_scal, scal.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, st()));
        OSMPM_CU(cudaStreamSynchronize(st()));
        return OSMPM_OK;
    }

    osmpm_status newton_gradient(const double* uin, double* gout, double* E, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        OSMPM_TRY(import_dense(uin, D, u.p, sp));
        OSMPM_TRY(grad_eval(u.p, false));
        if (gout) OSMPM_TRY(export_dense<double>(g.p, D, gout, sp));
        if (E) {
            OSMPM_TRY(read_scal(6));
            *E = (h_scal[2] > 0) ? INFINITY : h_scal[0] + h_scal[3];
        }
        return OSMPM_OK;
    }



    // HVP variant: sliding-window tiled kernel (default, hvp_sw.cuh); OSMPM_HVP=tiled | tiled_nopf | ws
    // select the earlier variants, kept for A/B measurements
    int hvp_variant() const
    {
        static int v = -1;
        if (v < 0) {
            const char* e = getenv("OSMPM_HVP");
            const std::string s = e ? e : "";
            v = (s == "ws") ? 1 : (s == "tiled_nopf") ? 2 : (s == "tiled") ? 0 : 3;
        }
        return v;
    }

    osmpm_status launch_hvp(const double* din, double* yout)
    {
        auto& pf = ctx->prof;
        if (pf.on) pf.begin("hvp", st());
        if (hvp_variant() == 1) {
            using Lay = WSLayout<D, R>;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_hvp_ws<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::BYTES);
                attr = true;
            }
            const int grid = std::max(1, std::min(box.ntiles, ctx->num_sms));
            KC(); k_hvp_ws<D, R><<<grid, WS<D>::NTHR, Lay::BYTES, st()>>>(P.p, cache.p, cap, cell_start.p, box, din,
                                                                          yout);
        } else if (hvp_variant() == 2) {
            static bool attr2 = false;
            if (!attr2) {
                cudaFuncSetAttribute(k_hvp<D, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)hvp_smem_bytes<D, R, false>());
                attr2 = true;
            }
            KC(); k_hvp<D, R, false><<<box.ntiles, T::NT, hvp_smem_bytes<D, R, false>(), st()>>>(
                P.p, cache.p, cap, cell_start.p, box, din, yout);
        } else if (hvp_variant() == 0) {
            KC(); k_hvp<D, R><<<box.ntiles, T::NT, hvp_smem(), st()>>>(P.p, cache.p, cap, cell_start.p, box, din, yout);
        } else {
            static bool attr3 = false;
            if (!attr3) {
                cudaFuncSetAttribute(k_hvp_sw<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)hvp_sw_smem_bytes<D, R>());
                attr3 = true;
            }
            KC(); k_hvp_sw<D, R><<<box.ntiles, T::NT, hvp_sw_smem_bytes<D, R>(), st()>>>(P.p, cache.p, cap,
                                                                                         cell_start.p, box, din, yout);
        }
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("hvp", st());
        return OSMPM_OK;
    }

    osmpm_status newton_hvp(const double* din, double* yout, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        if (!have_lin) {
            set_error("newton_hvp needs a prior newton_gradient (linearisation point)");
            return OSMPM_E_STATE;
        }
        const size_t nn = box.nnodes;
        OSMPM_TRY(import_dense(din, D, p.p, sp));
        OSMPM_CU(cudaMemsetAsync(y.p, 0, nn * D * sizeof(double), st()));
        OSMPM_TRY(launch_hvp(p.p, y.p));
        KC(); k_add_mass<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, m.p, 1.0 / (dt * dt), p.p, y.p);
        OSMPM_LAUNCH_CHECK();
        return export_dense<double>(y.p, D, yout, sp);
    }

    osmpm_status newton_diag(double* dout, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        if (!have_lin) {
            set_error("newton_diag needs a prior newton_gradient");
            return OSMPM_E_STATE;
        }
        return export_dense<double>(dg.p, D, dout, sp);
    }

    // =========================================================================================
    // a3-a7: Newton-PCG with backtracking line search
    // =========================================================================================
    osmpm_status build_dirichlet()
    {
        const size_t nn = box.nnodes;
        OSMPM_CU(cudaMemsetAsync(dmask.p, 0, nn, st()));
        OSMPM_CU(cudaMemsetAsync(dval.p, 0, nn * D * sizeof(double), st()));
        for (DirList* dl : {&dir_user, &dir_cpl})
            if (dl->n > 0) {
                KC(); k_scatter_dirichlet<D><<<nblk_all(dl->n, 256), 256, 0, st()>>>(box, dl->n, dl->idx.p, dl->mask.p,
                                                                               dl->val.p, dmask.p, dval.p);
                OSMPM_LAUNCH_CHECK();
            }
        return OSMPM_OK;
    }

    osmpm_status set_dirichlet(int64_t nd, const int64_t* idx, const uint8_t* mask, const double* vel,
                               osmpm_memspace sp) override
    {
        return set_dirlist(dir_user, nd, idx, mask, vel, sp);
    }

    osmpm_status set_dirlist(DirList& dl, int64_t nd, const int64_t* idx, const uint8_t* mask, const double* vel,
                             osmpm_memspace sp)
    {
        dl.n = nd;
        if (nd == 0) return OSMPM_OK;
        OSMPM_TRY(dl.idx.need(nd));
        OSMPM_TRY(dl.mask.need(nd));
        OSMPM_TRY(dl.val.need(nd * D));
        cudaMemcpyKind k = sp == OSMPM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        OSMPM_CU(cudaMemcpyAsync(dl.idx.p, idx, nd * sizeof(int64_t), k, st()));
        OSMPM_CU(cudaMemcpyAsync(dl.mask.p, mask, nd, k, st()));
        OSMPM_CU(cudaMemcpyAsync(dl.val.p, vel, nd * D * sizeof(double), k, st()));
        if (sp == OSMPM_HOST) OSMPM_CU(cudaStreamSynchronize(st()));
        return OSMPM_OK;
    }

    osmpm_status energy_eval(const double* uu)
    {
        const size_t nn = box.nnodes;
        auto& pf = ctx->prof;
        const int nbp = nblk(n, 256);
        if (pf.on) pf.begin("energy", st());
        KC(); k_energy<D, R><<<nbp, 256, 0, st()>>>(P.p, cap, n, mat.p, box, mats, uu, partA.p);
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("energy", st());
        const int nbn = nblk(nn, 256);
        KC(); k_energy_nodes<D><<<nbn, 256, 0, st()>>>(nn, m.p, vn.p, uu, dt, grav[0], grav[1], grav[2], partB.p);
        OSMPM_LAUNCH_CHECK();
        // scal[8..10] particles {E, E_abs, inverted}; scal[11..12] nodes {E, E_abs}
        KC(); k_final_sum<3><<<1, 1024, 0, st()>>>(partA.p, nbp, scal.p + 8);
        KC(); k_final_sum<2><<<1, 1024, 0, st()>>>(partB.p, nbn, scal.p + 11);
        OSMPM_LAUNCH_CHECK();
        return OSMPM_OK;
    }



    osmpm_status implicit_solve(const osmpm_newton_settings* s, osmpm_solve_stats* stats) override
    {
        OSMPM_TRY(need_grid());
        osmpm_solve_stats stl{};
        osmpm_solve_stats* sts = stats ? stats : &stl;
        std::memset(sts, 0, sizeof(*sts));
        const size_t nn = box.nnodes, ndof = nn * D;
        OSMPM_TRY(build_dirichlet());
        KC(); k_newton_init<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, act.p, dmask.p, dval.p, vn.p, dt, s->guess, fmask.p,
                                                               u.p);
        OSMPM_LAUNCH_CHECK();
        const double idt2 = 1.0 / (dt * dt);
        double g0 = 0.0, gref = 0.0;
        // E(u) for the line search comes from the same energy kernel as the trial energies, so both
        // sides of the comparison round alike (R8); later iterations reuse the accepted trial
        double E0n = 0.0, Ea0n = 0.0;
        if (s->max_newton > 0) {
            OSMPM_TRY(energy_eval(u.p));
            OSMPM_TRY(read_scal(13));
            E0n = (h_scal[10] > 0) ? INFINITY : h_scal[8] + h_scal[11];
            Ea0n = h_scal[9] + h_scal[12];
        }
        bool converged = false;
        osmpm_status rc = OSMPM_OK;
        const int nbd = nblk(ndof, 256), nbn = nblk(nn, 256);
        const int chunk = s->fixed_iters ? s->max_cg : 8;
        for (int it = 0; it < s->max_newton; ++it) {
            OSMPM_TRY(grad_eval(u.p, true));
            OSMPM_TRY(read_scal(7));
            const double gn = std::sqrt(h_scal[5]);
            const double E0 = E0n, Ea0 = Ea0n;
            if (it == 0) {
                // Newton test relative to max(|g^(0)|, force scale) (R6)
                g0 = gn;
                gref = std::max(g0, std::sqrt(h_scal[6]));
            }
            sts->grad_norm = gn;
            if (!s->fixed_iters && (gn <= s->newton_rtol * gref || gn <= s->newton_atol)) {
                converged = true;
                break;
            }
            // Jacobi PCG on H dx = -g (R6, R7)
            KC(); k_cg_init<D><<<nbd, 256, 0, st()>>>(ndof, fmask.p, g.p, dg.p, r.p, z.p, p.p, xs.p, y.p, partB.p);
            KC(); k_cg_init_fin<<<1, 1024, 0, st()>>>(partB.p, nbd, cgs.p, gn, s->cg_rtol, s->fixed_iters);
            OSMPM_LAUNCH_CHECK();
            int done_it = 0;
            while (done_it < s->max_cg) {
                const int cnt = std::min(chunk, s->max_cg - done_it);
                for (int c = 0; c < cnt; ++c) {
                    OSMPM_TRY(launch_hvp(p.p, y.p));
                    if (ctx->prof.on) ctx->prof.begin("cg", st());
                    KC(); k_cg_q<D><<<nbn, 256, 0, st()>>>(nn, fmask.p, m.p, idt2, p.p, y.p, cgs.p, partB.p);
                    KC(); k_cg_alpha<<<1, 1024, 0, st()>>>(partB.p, nbn, cgs.p);
                    KC(); k_cg_update<<<nbd, 256, 0, st()>>>(ndof, fmask.p, p.p, y.p, dg.p, xs.p, r.p, z.p, cgs.p, partB.p);
                    KC(); k_cg_beta<<<1, 1024, 0, st()>>>(partB.p, nbd, cgs.p);
                    KC(); k_cg_p<<<nbd, 256, 0, st()>>>(ndof, z.p, p.p, y.p, cgs.p);
                    if (ctx->prof.on) ctx->prof.end("cg", st());
                    OSMPM_LAUNCH_CHECK();
                }
                done_it += cnt;
                if (!s->fixed_iters) {
                    OSMPM_CU(cudaMemcpyAsync(h_cgs, cgs.p, sizeof(CGScalars), cudaMemcpyDeviceToHost, st()));
                    OSMPM_CU(cudaStreamSynchronize(st()));
                    if (h_cgs->done) break;
                }
            }
            OSMPM_CU(cudaMemcpyAsync(h_cgs, cgs.p, sizeof(CGScalars), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            sts->cg_iters += h_cgs->it + (h_cgs->done == 2 ? 1 : 0);
            if (h_cgs->negcurv_first) OSMPM_CU(cudaMemcpyAsync(xs.p, z.p, ndof * sizeof(double), cudaMemcpyDeviceToDevice, st()));
            // backtracking line search (R8)
            double alpha = 1.0, Et = 0.0, Eat = 0.0;
            for (;;) {
                KC(); k_axpy_free<<<nbd, 256, 0, st()>>>(ndof, fmask.p, u.p, alpha, xs.p, ut.p);
                OSMPM_LAUNCH_CHECK();
                OSMPM_TRY(energy_eval(ut.p));
                OSMPM_TRY(read_scal(13));
                const bool inv = h_scal[10] > 0;
                Et = inv ? INFINITY : h_scal[8] + h_scal[11];
                Eat = h_scal[9] + h_scal[12];
                if (Et < E0 || (std::isfinite(Et) && std::fabs(Et - E0) <= s->energy_noise_rtol * Ea0)) break;
                alpha *= 0.5;
                sts->ls_halvings++;
                if (alpha < s->ls_min_alpha) {
                    set_error("line search stagnated at Newton iteration %d (alpha < %g)", it, s->ls_min_alpha);
                    rc = OSMPM_E_LINESEARCH_STAGNATION;
                    break;
                }
            }
            if (rc != OSMPM_OK) break;
            std::swap(u.p, ut.p);
            std::swap(u.cap, ut.cap);
            E0n = Et;
            Ea0n = Eat;
            sts->energy = Et;
            sts->newton_iters = it + 1;
        }
        if (rc == OSMPM_OK && !s->fixed_iters && !converged) {
            OSMPM_TRY(grad_eval(u.p, true));
            OSMPM_TRY(read_scal(6));
            const double gn = std::sqrt(h_scal[5]);
            sts->grad_norm = gn;
            if (!(gn <= s->newton_rtol * gref || gn <= s->newton_atol)) {
                set_error("Newton did not converge in %d iterations (|g| = %g, |g0| = %g)", s->max_newton, gn, g0);
                rc = OSMPM_E_NEWTON_NOT_CONVERGED;
            }
        }
        sts->grad_norm0 = g0;
        sts->status = rc;
        KC(); k_vnew<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, act.p, u.p, 1.0 / dt, vnew.p);
        OSMPM_LAUNCH_CHECK();
        have_vnew = true;
        have_lin = false;  // the cache now refers to an intermediate point
        return rc;
    }

    osmpm_status read_grid_velocity(double* v, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        if (!have_vnew) {
            set_error("no solved grid velocity");
            return OSMPM_E_STATE;
        }
        return export_dense<double>(vnew.p, D, v, sp);
    }
    osmpm_status set_grid_velocity(const double* v, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        OSMPM_TRY(import_dense(v, D, vnew.p, sp));
        have_vnew = true;
        return OSMPM_OK;
    }

    // =========================================================================================
    // a8: G2P
    // =========================================================================================
    osmpm_status g2p() override
    {
        OSMPM_TRY(need_grid());
        if (!have_vnew) {
            set_error("osmpm_g2p needs a solved (or set) grid velocity");
            return OSMPM_E_STATE;
        }
        auto& pf = ctx->prof;
        if (pf.on) pf.begin("g2p", st());
        if (n > 0) {
            KC(); k_g2p<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, pid.p, box, vnew.p, dt, err.p);
            OSMPM_LAUNCH_CHECK();
        }
        if (pf.on) pf.end("g2p", st());
        have_grid = false;  // particles moved: the next step starts with P2G
        have_lin = false;
        have_vnew = false;
        return OSMPM_OK;
    }

    // =========================================================================================
    // particle I/O (creation order)
    // =========================================================================================
    osmpm_status read_particles(double* x, double* v, double* F, double* B, osmpm_memspace sp) override
    {
        struct Fld { double* dst; int off, nc; };
        const Fld flds[] = {{x, L::X, D}, {v, L::V, D}, {F, L::F, D * D}, {B, L::B, D * D}};
        for (const Fld& fl : flds) {
            if (!fl.dst || n == 0) continue;
            const size_t cnt = (size_t)n * fl.nc;
            double* d = fl.dst;
            DBuf<double>& stage = stage_io;
            if (sp == OSMPM_HOST) {
                OSMPM_TRY(stage.need(cnt));
                d = stage.p;
            }
            for (int c = 0; c < fl.nc; ++c) {
                KC(); k_unsort_field<R><<<nblk_all(n, 256), 256, 0, st()>>>(P.p + (size_t)(fl.off + c) * cap, n, pid.p,
                                                                      fl.nc, c, d);
            }
            OSMPM_LAUNCH_CHECK();
            if (sp == OSMPM_HOST) {
                OSMPM_CU(cudaMemcpyAsync(fl.dst, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, st()));
                OSMPM_CU(cudaStreamSynchronize(st()));
            }
        }
        return OSMPM_OK;
    }

    osmpm_status set_particles(const double* x, const double* v, const double* F, const double* B,
                               osmpm_memspace sp) override
    {
        struct Fld { const double* src; int off, nc; };
        const Fld flds[] = {{x, L::X, D}, {v, L::V, D}, {F, L::F, D * D}, {B, L::B, D * D}};
        for (const Fld& fl : flds) {
            if (!fl.src || n == 0) continue;
            const size_t cnt = (size_t)n * fl.nc;
            const double* s = fl.src;
            DBuf<double>& stage = stage_io;
            if (sp == OSMPM_HOST) {
                OSMPM_TRY(stage.need(cnt));
                OSMPM_CU(cudaMemcpyAsync(stage.p, fl.src, cnt * sizeof(double), cudaMemcpyHostToDevice, st()));
                s = stage.p;
            }
            for (int c = 0; c < fl.nc; ++c) {
                KC(); k_sort_field<R><<<nblk_all(n, 256), 256, 0, st()>>>(s, n, pid.p, fl.nc, c,
                                                                    P.p + (size_t)(fl.off + c) * cap);
            }
            OSMPM_LAUNCH_CHECK();
            if (sp == OSMPM_HOST) OSMPM_CU(cudaStreamSynchronize(st()));
        }
        have_grid = have_lin = have_vnew = false;
        return OSMPM_OK;
    }

    osmpm_status info(int64_t* np, int64_t* lo, int64_t* dims) override
    {
        if (np) *np = n;
        for (int a = 0; a < 3; ++a) {
            if (lo) lo[a] = box.lo[a];
            if (dims) dims[a] = box.nn[a];
        }
        return OSMPM_OK;
    }

    // checkpoint / restore of the whole particle state (K11)
    osmpm_status checkpoint()
    {
        OSMPM_TRY(Pck.need(L::NF * cap));
        OSMPM_TRY(matck.need(cap));
        OSMPM_TRY(pidck.need(cap));
        OSMPM_TRY(bndck.need(cap));
        OSMPM_CU(cudaMemcpyAsync(Pck.p, P.p, (size_t)L::NF * cap * sizeof(R), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(matck.p, mat.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(pidck.p, pid.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(bndck.p, bnd.p, cap, cudaMemcpyDeviceToDevice, st()));
        have_ck = true;
        return OSMPM_OK;
    }
    osmpm_status restore()
    {
        if (!have_ck) {
            set_error("restore without checkpoint");
            return OSMPM_E_STATE;
        }
        OSMPM_CU(cudaMemcpyAsync(P.p, Pck.p, (size_t)L::NF * cap * sizeof(R), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(mat.p, matck.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(pid.p, pidck.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(bnd.p, bndck.p, cap, cudaMemcpyDeviceToDevice, st()));
        have_grid = have_lin = have_vnew = false;
        return OSMPM_OK;
    }
};

}  // namespace osmpm
