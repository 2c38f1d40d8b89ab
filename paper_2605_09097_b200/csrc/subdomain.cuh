// subdomain.cuh -- one MPM subdomain on one GPU (§3.1: its own grid dx, time step dt and
// particle set), templated on dimension D and particle precision R.
#pragma once

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "radix_sort.cuh"
#include "psd.cuh"
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

// Scalar / reduction buffers of a slab group (one standalone subdomain = a group of one slab).
// Block partials of every slab of the group are laid out back to back in partA / partB so that ONE
// fixed-order final sum reduces the whole group (deterministic); across ranks the sums are
// ncclAllReduce'd before use.
struct CGScalars;
// Host state of the fused HVP halo (R24, hvp_sw.cuh HaloDev): per-slab CTA completion
// counters, this rank's inbox words (bumped by the neighbouring ranks' HVPs) and the neighbouring
// ranks' y buffers and inboxes mapped over NVLink with CUDA IPC (cached by handle).
struct HaloPeer {
    static constexpr int NB = 3;  // y at the exchange, its double buffer, the inbox words
    cudaIpcMemHandle_t h[NB];
    void* p[NB] = {nullptr, nullptr, nullptr};
    int64_t nn0 = 0;  // x node planes of the peer's box (its slab next to this rank)
    void close()
    {
        for (int k = 0; k < NB; ++k)
            if (p[k]) cudaIpcCloseMemHandle(p[k]);
        for (int k = 0; k < NB; ++k) p[k] = nullptr;
    }
};
struct HaloLink {  // one side of a local slab
    double* y[2] = {nullptr, nullptr};  // alternating protocol: the neighbour's y / y2 at the setup
    unsigned* sig = nullptr;            // the neighbour's inbox word this slab bumps
    int64_t nn0 = 0;                    // the neighbour's x node planes
    bool on = false;                    // the protocol runs on this side (else: plain pointer or none)
};
struct HaloState {
    DBuf<unsigned> done;   // one completion counter per local slab (zero between launches)
    DBuf<unsigned> inbox;  // per local slab: [2i] bumped by the left neighbour, [2i + 1] by the right one
    int ndone = 0;
    bool alt = false;      // some side runs the alternating protocol in this solve
    unsigned rounds = 0;   // protocol HVP rounds since the inbox words were zeroed
    int phase = 0;         // y / y2 swaps since the setup (selects the neighbours' buffer)
    std::vector<HaloLink> L, R;
    HaloPeer left, right;
    ~HaloState()
    {
        left.close();
        right.close();
    }
};
struct GroupBufs {
    DBuf<double> partA, partB, partH, scal, gsum, halo_tmp;  // partH: the HVP's d^T K d partials (R22)
    DBuf<CGScalars> cgs;
    DBuf<unsigned> tick;  // last-block tickets of k_cg_q_alpha / k_cg_update_beta (reset by the last block)
    DBuf<int> gbounds;
    HaloState halo;
    double* h_scal = nullptr;  // pinned
    CGScalars* h_cgs = nullptr;
    int* h_bounds = nullptr;
    osmpm_status init()
    {
        if (h_scal) return OSMPM_OK;
        OSMPM_CU(cudaMallocHost((void**)&h_scal, 64 * sizeof(double)));
        OSMPM_CU(cudaMallocHost((void**)&h_cgs, 256));
        OSMPM_CU(cudaMallocHost((void**)&h_bounds, 8 * sizeof(int)));
        OSMPM_TRY(scal.need(64));
        OSMPM_TRY(gsum.need(8));
        OSMPM_TRY(cgs.need(1));
        OSMPM_TRY(tick.need(2));
        OSMPM_CU(cudaMemset(tick.p, 0, 2 * sizeof(unsigned)));
        OSMPM_TRY(gbounds.need(8));
        return OSMPM_OK;
    }
    ~GroupBufs()
    {
        if (h_scal) cudaFreeHost(h_scal);
        if (h_cgs) cudaFreeHost(h_cgs);
        if (h_bounds) cudaFreeHost(h_bounds);
    }
};

template <int D, typename R> struct Sub;
template <int D, typename R> struct SlabGroup {
    Sub<D, R>* const* s;  // local slabs, ordered along x
    int ns;
    GroupComm* gc;        // nullptr or no communicator: no inter-rank exchange
    GroupBufs* gb;
    cudaStream_t st;
    osmpm_ctx* ctx;
    bool multi() const { return gc && gc->multi(); }
};
template <int D, typename R> osmpm_status group_p2g(SlabGroup<D, R> G);
template <int D, typename R> osmpm_status group_grad(SlabGroup<D, R> G, bool need_fmask, bool trial = false);
template <int D, typename R> osmpm_status group_energy(SlabGroup<D, R> G, bool trial);
template <int D, typename R> osmpm_status group_solve(SlabGroup<D, R> G, const osmpm_newton_settings* s,
                                                      osmpm_solve_stats* stats);
template <int D, typename R> osmpm_status group_hvp(SlabGroup<D, R> G);

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
    DBuf<uint32_t> rs_hist;  // digit histograms of the radix sort (radix_sort.cuh)

    // ---- node box ---------------------------------------------------------------------------
    BoxDev box{};
    bool have_grid = false, have_lin = false, have_vnew = false, have_vlast = false;
    DBuf<int> cell_start;
    DBuf<double> m, mom, vn, fsig, mb, dval, u, g, dg, xs, r, z, p, y, ut, vnew, tmp, cs;  // cs: s = H p (R22)
    DBuf<double> y2;  // second HVP output buffer, alternated with y between ranks (fused halo, R24)
    DBuf<uint8_t> act, dmask, fmask;
    DirList dir_user, dir_cpl;
    DBuf<double> stage_io;  // persistent host-I/O staging buffer
    DBuf<int> pi_gd;  // dense-box dims on the device when this subdomain is Pi's coarse side (transmit.cuh)
    DBuf<double> Tpsd;        // PSD-projected tangent blocks (psd.cuh), packed, field-major
    bool psd_active = false;  // the HVP of the current PCG solve uses them (R23)
    DBuf<double> det_a, det_b, det_c;  // per-tile node blocks of the deterministic scatter mode (hvp_sw.cuh)

    // OSMPM_DETERMINISTIC=1: the sliding-window gradient and HVP store per-tile node blocks that a
    // node pass sums in a fixed tile order instead of RED-ing into the node arrays (bitwise
    // reproducible Newton-PCG; read at every launch so a process can switch)
    // det_force: set by the coupler on the replicated coarse subdomain of a multi-rank run, so that every
    // rank computes bitwise the same coarse solution
    bool det_force = false;
    bool det_mode() const
    {
        const char* e = getenv("OSMPM_DETERMINISTIC");
        return det_force || (e && e[0] == '1');
    }
    osmpm_status det_gather(const double* tb, double* out)
    {
        KC(); k_det_gather<D><<<nblk_all(box.nnodes, 256), 256, 0, st()>>>(box, cell_start.p, tb, out);
        OSMPM_LAUNCH_CHECK();
        return OSMPM_OK;
    }

    // ---- reductions / scalars ---------------------------------------------------------------
    GroupBufs gbself;  // used when the subdomain is standalone (a group of one slab)
    DBuf<ErrLatch> err;
    DBuf<int> bounds;
    int* h_bounds = nullptr;
    int part_off = 0;  // this slab's block-partial offset inside its group's partial buffers
    CUtensorMap tm_x{}, tm_c{};  // HVP streamed-input tensor maps (hvp_sw.cuh) and what they describe
    const void* tm_P = nullptr;
    const void* tm_C = nullptr;
    int64_t tm_cap = -1;
    bool tm_ok = false;

    // ---- slab decomposition --------------------------------------------------
    // cells [cut_lo, cut_hi) along x (INT32_MIN / INT32_MAX: open end).  A slab with a right
    // neighbour carries the neighbour's first two node planes as ghosts (the last two planes of its
    // box, x being the slowest box axis): scatters into them are reverse-added to the owner, and the
    // owner's sums copied back, so every node array is consistent on owners and ghosts.
    int cut_lo = INT32_MIN, cut_hi = INT32_MAX;
    bool ghost_right = false;
    int64_t nown = 0;  // owned box nodes (all but the ghost planes)

    ~Sub() override
    {
        if (h_bounds) cudaFreeHost(h_bounds);
    }

    SlabGroup<D, R> self_group()
    {
        Sub<D, R>* const* me = &self_ptr;
        self_ptr = this;
        return SlabGroup<D, R>{me, 1, nullptr, &gbself, st(), ctx};
    }
    Sub<D, R>* self_ptr = nullptr;

    cudaStream_t st() const { return ctx->stream; }
    void KC() const { ctx->launches++; }

    // =========================================================================================
    // creation
    // =========================================================================================
    // sel: the creation indices of the particles this subdomain (slab) takes (nullptr: all of them);
    // cap_min: particle capacity to reserve (slabs keep slack for migration)
    osmpm_status create(const osmpm_grid_desc* gd, double dt_, const osmpm_particles_view* pv,
                        const osmpm_material* mt, int nm, const double* gravity, const int64_t* sel = nullptr,
                        int64_t nsel = -1, int64_t cap_min = 0)
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
        n = sel ? nsel : pv->n;
        const int64_t nall = pv->n;
        auto src_of = [&](int64_t i) -> int64_t { return sel ? sel[i] : i; };
        // field stride: a multiple of 4 (16-B aligned fields for the TMA bulk copies) with >= 4
        // elements of slack (bulk copies round their length up to 16 B)
        cap = ((std::max(n, cap_min) + 4 + 3) / 4) * 4;
        OSMPM_TRY(gbself.init());
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
            const double* s = host_view(fl.src, (size_t)nall * fl.nc);
            for (int c = 0; c < fl.nc; ++c)
                for (int64_t i = 0; i < n; ++i) {
                    double v = s ? s[src_of(i) * fl.nc + c] : 0.0;
                    if (!s && fl.off == L::F && (c % (D + 1)) == 0) v = 1.0;
                    h[(size_t)(fl.off + c) * cap + i] = (R)v;
                }
        }
        if (pv->material) {
            std::vector<int> all(nall);
            if (pv->space == OSMPM_HOST)
                std::memcpy(all.data(), pv->material, nall * sizeof(int));
            else
                cudaMemcpy(all.data(), pv->material, nall * sizeof(int), cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < n; ++i) {
                hm[i] = all[src_of(i)];
                if (hm[i] < 0 || hm[i] >= nm) {
                    set_error("particle %lld: material %d outside [0, %d)", (long long)src_of(i), hm[i], nm);
                    return OSMPM_E_INVALID_ARG;
                }
            }
        }
        if (pv->is_boundary) {
            std::vector<uint8_t> all(nall);
            if (pv->space == OSMPM_HOST)
                std::memcpy(all.data(), pv->is_boundary, nall);
            else
                cudaMemcpy(all.data(), pv->is_boundary, nall, cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < n; ++i) hb[i] = all[src_of(i)];
        }
        for (int64_t i = 0; i < n; ++i) hp[i] = (int)src_of(i);
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
        if (!sel) {
            OSMPM_TRY(compute_box());
            return check_err();
        }
        return OSMPM_OK;
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
            if (h.code == OSMPM_E_INVALID_ARG)
                set_error("transmit target %lld outside the destination node box", h.index);
            else if (h.code == OSMPM_E_OUT_OF_DOMAIN)
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

    // lowest / highest base node per axis of this subdomain's particles (and the safe-interior
    // check); INT32_MAX / INT32_MIN when it holds none
    osmpm_status bounds_local(int* lo, int* hi)
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
        for (int a = 0; a < 3; ++a) {
            lo[a] = h_bounds[a];
            hi[a] = h_bounds[3 + a];
        }
        return OSMPM_OK;
    }

    // node box of the step from the GROUP's base-node bounds glo / ghi (whole tiles; the x range of
    // a slab is its cut range, so neighbouring slabs share node planes exactly)
    void set_box(const int* glo, const int* ghi)
    {
        BoxDev b{};
        fill_box_common(b);
        const int tt[3] = {T::T0, T::T1, T::T2};
        const bool any = glo[0] <= ghi[0];
        int64_t ncells = 1, nnodes = 1;
        int ntiles = 1;
        for (int a = 0; a < 3; ++a) {
            int lo = 0, c = tt[a];
            if (a < D && any) {
                lo = glo[a];
                int hiex = ghi[a] + 1;
                if (a == 0 && cut_lo != INT32_MIN) lo = cut_lo;
                if (a == 0 && cut_lo == INT32_MIN && cut_hi != INT32_MAX) {
                    // first slab: align down from the first cut so that the cut is a tile boundary
                    const int w = std::max(cut_hi - glo[0], 1);
                    lo = cut_hi - ((w + tt[0] - 1) / tt[0]) * tt[0];
                }
                if (a == 0 && cut_hi != INT32_MAX) hiex = cut_hi;
                c = std::max(hiex - lo, 1);
                c = ((c + tt[a] - 1) / tt[a]) * tt[a];
            } else if (a >= D) {
                c = 1;
            }
            b.lo[a] = lo;
            b.nc[a] = c;
            b.nn[a] = (a < D) ? c + 2 : 1;
            b.nt[a] = (a < D) ? c / tt[a] : 1;
            ncells *= b.nc[a];
            nnodes *= b.nn[a];
            ntiles *= b.nt[a];
        }
        b.ncells = ncells;
        b.nnodes = nnodes;
        b.ntiles = ntiles;
        box = b;
        ghost_right = cut_hi != INT32_MAX;
        const int64_t plane = (D == 3) ? (int64_t)b.nn[1] * b.nn[2] : b.nn[1];
        nown = ghost_right ? nnodes - 2 * plane : nnodes;
    }
    int64_t plane_nodes() const { return (D == 3) ? (int64_t)box.nn[1] * box.nn[2] : box.nn[1]; }

    osmpm_status compute_box()
    {
        int lo[3], hi[3];
        OSMPM_TRY(bounds_local(lo, hi));
        set_box(lo, hi);
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
        KC(); k_keys<D, R><<<nblk_all(n, 256), 256, 0, st()>>>(P.p, cap, n, box, keys.p, vals.p, pid.p, err.p);
        OSMPM_LAUNCH_CHECK();
        int nbits = 1;
        while ((int64_t(1) << nbits) < box.ncells) ++nbits;
        OSMPM_TRY(rs_hist.need(radix_hist_words(n)));
        // stable LSD radix sort of the cell keys (radix_sort.cuh); the sorted pairs end in keys2/vals2
        if (!radix_sort_pairs(keys.p, vals.p, keys2.p, vals2.p, n, nbits, rs_hist.p, st(), ctx->launches)) {
            std::swap(keys.p, keys2.p);
            std::swap(keys.cap, keys2.cap);
            std::swap(vals.p, vals2.p);
            std::swap(vals.cap, vals2.cap);
        }
        OSMPM_LAUNCH_CHECK();
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
        for (DBuf<double>* b : {&mom, &vn, &fsig, &dval, &u, &g, &dg, &xs, &r, &z, &p, &y, &ut, &vnew, &cs})
            OSMPM_TRY(b->need(nd));
        OSMPM_TRY(act.need(nn));
        OSMPM_TRY(dmask.need(nn));
        OSMPM_TRY(fmask.need(nd));
        return OSMPM_OK;
    }

    // =========================================================================================
    // a2: P2G
    // =========================================================================================
    // P2G of this slab: sort, scatter (the group then halo-sums m, mom, f^sigma), node pass
    osmpm_status p2g_scatter()
    {
        OSMPM_TRY(sort_particles());
        OSMPM_TRY(alloc_nodes());
        const size_t nn = box.nnodes;
        OSMPM_CU(cudaMemsetAsync(m.p, 0, nn * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(mom.p, 0, nn * D * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(fsig.p, 0, nn * D * sizeof(double), st()));
        if (n > 0) {
            // tiled P2G (p2g_tiled.cuh)
            {
                static bool attr = false;
                if (!attr) {
                    cudaFuncSetAttribute(k_p2g_tiled<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p2g_tiled_smem_bytes<D, R>());
                    attr = true;
                }
                const bool det = det_mode();
                if (det) {
                    OSMPM_TRY(det_a.need((size_t)box.ntiles * T::NN * D));
                    OSMPM_TRY(det_b.need((size_t)box.ntiles * T::NN * D));
                    OSMPM_TRY(det_c.need((size_t)box.ntiles * T::NN));
                }
                KC(); k_p2g_tiled<D, R><<<box.ntiles, T::NT, p2g_tiled_smem_bytes<D, R>(), st()>>>(
                    P.p, cap, mat.p, cell_start.p, box, mats, m.p, mom.p, fsig.p, det ? det_c.p : nullptr,
                    det ? det_a.p : nullptr, det ? det_b.p : nullptr);
                if (det) {
                    OSMPM_LAUNCH_CHECK();
                    KC(); k_det_gather<D, 1><<<nblk_all(box.nnodes, 256), 256, 0, st()>>>(box, cell_start.p, det_c.p, m.p);
                    OSMPM_TRY(det_gather(det_a.p, mom.p));
                    OSMPM_TRY(det_gather(det_b.p, fsig.p));
                }
            }
            OSMPM_LAUNCH_CHECK();
        }
        return OSMPM_OK;
    }
    osmpm_status p2g_nodes()
    {
        const size_t nn = box.nnodes;
        KC(); k_p2g_nodes<D><<<nblk_all(nn, 256), 256, 0, st()>>>(nn, m.p, mom.p, vn.p, act.p, mass_thr);
        OSMPM_LAUNCH_CHECK();
        have_grid = true;
        have_lin = false;
        have_vnew = false;
        have_vlast = false;
        return OSMPM_OK;
    }
    osmpm_status p2g() override { return group_p2g<D, R>(self_group()); }

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
        if (have_grid || have_vlast) {  // have_vlast: the box of the last P2G is still the current one
            KC(); k_box_to_dense<D, Tv><<<nblk_all(box.nnodes, 256), 256, 0, st()>>>(box, nown, nc, src, dptr);
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
    // a4: gradient + energy at u (box vector) -> g (raw), dg (raw); block partials into the group's
    // buffers: particle part {E, |E|, inverted} (partA), node part {E, |E|, |g_free|^2, f_scale^2}
    // (partB, owned nodes only)
    // =========================================================================================
    int grad_blocks_nodes() const { return nblk(box.nnodes, 256); }

    osmpm_status grad_scatter(const double* uu, bool need_fmask, double* partA)
    {
        const size_t nn = box.nnodes;
        OSMPM_TRY(cache.need(C::NF * cap));
        OSMPM_CU(cudaMemsetAsync(g.p, 0, nn * D * sizeof(double), st()));
        OSMPM_CU(cudaMemsetAsync(dg.p, 0, nn * D * sizeof(double), st()));
        if (!need_fmask) OSMPM_CU(cudaMemsetAsync(fmask.p, 1, nn * D, st()));
        // sliding-window gradient (grad_sw.cuh)
        static bool attr_sw = false;
        if (!attr_sw) {
            cudaFuncSetAttribute(k_grad_sw<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)grad_sw_smem_bytes<D, R>());
            attr_sw = true;
        }
        const bool det = det_mode();
        if (det) {
            OSMPM_TRY(det_a.need((size_t)box.ntiles * T::NN * D));
            OSMPM_TRY(det_b.need((size_t)box.ntiles * T::NN * D));
        }
        KC(); k_grad_sw<D, R><<<box.ntiles, T::NT, grad_sw_smem_bytes<D, R>(), st()>>>(
            P.p, cache.p, cap, mat.p, cell_start.p, box, mats, uu, g.p, dg.p, partA, det ? det_a.p : nullptr,
            det ? det_b.p : nullptr);
        OSMPM_LAUNCH_CHECK();
        if (det) {
            OSMPM_TRY(det_gather(det_a.p, g.p));
            OSMPM_TRY(det_gather(det_b.p, dg.p));
        }
        return OSMPM_OK;
    }
    osmpm_status grad_nodes(const double* uu, double* partB)
    {
        KC(); k_grad_nodes<D><<<grad_blocks_nodes(), 256, 0, st()>>>(box.nnodes, nown, m.p, vn.p, uu, fmask.p, dt, grav[0],
                                                                      grav[1], grav[2], g.p, dg.p, partB);
        OSMPM_LAUNCH_CHECK();
        have_lin = true;
        return OSMPM_OK;
    }

    osmpm_status newton_gradient(const double* uin, double* gout, double* E, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        OSMPM_TRY(import_dense(uin, D, u.p, sp));
        auto G = self_group();
        OSMPM_TRY(group_grad<D, R>(G, false));
        if (gout) OSMPM_TRY(export_dense<double>(g.p, D, gout, sp));
        if (E) *E = (gbself.h_scal[2] > 0) ? INFINITY : gbself.h_scal[0] + gbself.h_scal[3];
        return OSMPM_OK;
    }

    // a5: the sliding-window tiled HVP (hvp_sw.cuh)
    // halo (optional): the fused halo of a slab group (R24); only the tiled fp64/fp32 kernel carries it
    // (the caller falls back to halo_sum when psd_active or in deterministic mode)
    osmpm_status launch_hvp(const double* din, double* yout, double* pkp = nullptr, const HaloDev* halo = nullptr)
    {
        auto& pf = ctx->prof;
        if (pf.on) pf.begin("hvp", st());
        if (psd_active) {
            // projected-tangent variant (psd.cuh): per-particle scatter; the single-reduction PCG's
            // curvature partials are not produced here, so psd solves use the standard PCG
            if (n > 0) {
                KC(); k_hvp_psd<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, box, Tpsd.p, din, yout);
            }
            OSMPM_LAUNCH_CHECK();
            if (pf.on) pf.end("hvp", st());
            return OSMPM_OK;
        }
        static bool attr3 = false;
        if (!attr3) {
            cudaFuncSetAttribute(k_hvp_sw<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)hvp_sw_smem_bytes<D, R>());
            attr3 = true;
        }
        // tensor maps of the streamed inputs, re-encoded when a buffer moves (the sort swaps P); if the
        // driver's encoder is unavailable the kernel streams the fields with per-field bulk copies
        if (tm_P != P.p || tm_C != cache.p || tm_cap != cap) {
            tm_ok = encode_fields_map<R>(&tm_x, P.p + (size_t)PL<D>::X * cap, D, cap, SWIn<D, R>::PFS) &&
                    encode_fields_map<R>(&tm_c, cache.p, C::NF, cap, SWIn<D, R>::PFS);
            tm_P = P.p;
            tm_C = cache.p;
            tm_cap = cap;
        }
        const bool det = det_mode();
        if (det) OSMPM_TRY(det_a.need((size_t)box.ntiles * T::NN * D));
        KC(); k_hvp_sw<D, R><<<box.ntiles, HvpT<D>::NT, hvp_sw_smem_bytes<D, R>(), st()>>>(
            P.p, cache.p, cap, cell_start.p, box, din, yout, tm_x, tm_c, tm_ok ? 1 : 0, det ? det_a.p : nullptr, pkp,
            (halo && !det) ? *halo : HaloDev{});
        if (det) {
            OSMPM_LAUNCH_CHECK();
            OSMPM_TRY(det_gather(det_a.p, yout));
        }
        OSMPM_LAUNCH_CHECK();
        if (pf.on) pf.end("hvp", st());
        return OSMPM_OK;
    }

    // R23: projected tangents at the current u, and the Jacobi diagonal they give (particle part; the
    // group adds the halo and the mass term)
    osmpm_status psd_scatter()
    {
        OSMPM_TRY(Tpsd.need((size_t)PSD<D>::NP * cap));
        OSMPM_CU(cudaMemsetAsync(dg.p, 0, box.nnodes * D * sizeof(double), st()));
        if (n > 0) {
            KC(); k_psd_tangent<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, mat.p, box, mats, u.p, Tpsd.p);
            KC(); k_diag_psd<D, R><<<nblk_all(n, 128), 128, 0, st()>>>(P.p, cap, n, box, Tpsd.p, dg.p);
        }
        OSMPM_LAUNCH_CHECK();
        return OSMPM_OK;
    }

    osmpm_status newton_hvp(const double* din, double* yout, osmpm_memspace sp) override
    {
        OSMPM_TRY(need_grid());
        if (!have_lin) {
            set_error("newton_hvp needs a prior newton_gradient (linearisation point)");
            return OSMPM_E_STATE;
        }
        OSMPM_TRY(import_dense(din, D, p.p, sp));
        OSMPM_TRY(group_hvp<D, R>(self_group()));
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

    // line-search energy at uu: block partials particle {E, |E|, inverted} (partA), node {E, |E|}
    // (partB, owned nodes only)
    // tiled (k_energy_tiled, one CTA per tile)
    int energy_blocks_particles() const { return box.ntiles; }
    osmpm_status energy_launch(const double* uu, double* partA, double* partB)
    {
        KC(); k_energy_tiled<D, R><<<box.ntiles, T::NT, 0, st()>>>(P.p, cap, mat.p, cell_start.p, box, mats, uu,
                                                                    partA);
        OSMPM_LAUNCH_CHECK();
        KC(); k_energy_nodes<D><<<grad_blocks_nodes(), 256, 0, st()>>>(box.nnodes, nown, m.p, vn.p, uu, dt, grav[0],
                                                                        grav[1], grav[2], partB);
        OSMPM_LAUNCH_CHECK();
        return OSMPM_OK;
    }

    osmpm_status implicit_solve(const osmpm_newton_settings* s, osmpm_solve_stats* stats) override
    {
        OSMPM_TRY(need_grid());
        return group_solve<D, R>(self_group(), s, stats);
    }

    osmpm_status read_grid_velocity(double* v, osmpm_memspace sp) override
    {
        if (!have_vlast) {
            OSMPM_TRY(need_grid());
            if (!have_vnew) {
                set_error("no solved grid velocity");
                return OSMPM_E_STATE;
            }
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
        have_vlast = true;  // vnew stays readable (the velocity the particles moved with) until the next P2G
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
        have_grid = have_lin = have_vnew = have_vlast = false;
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

    // checkpoint / restore of the whole particle state (K11).  The slab's
    // particle count is part of the state (migration changes it); the capacity never changes.
    int64_t n_ck = 0;
    osmpm_status checkpoint() override
    {
        n_ck = n;
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
    osmpm_status restore() override
    {
        if (!have_ck) {
            set_error("restore without checkpoint");
            return OSMPM_E_STATE;
        }
        n = n_ck;
        OSMPM_CU(cudaMemcpyAsync(P.p, Pck.p, (size_t)L::NF * cap * sizeof(R), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(mat.p, matck.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(pid.p, pidck.p, cap * sizeof(int), cudaMemcpyDeviceToDevice, st()));
        OSMPM_CU(cudaMemcpyAsync(bnd.p, bndck.p, cap, cudaMemcpyDeviceToDevice, st()));
        have_grid = have_lin = have_vnew = have_vlast = false;
        return OSMPM_OK;
    }
};

}  // namespace osmpm
