// coupler.cuh -- multiplicative Schwarz coupling of a coarse (B) and a fine (S) subdomain
// (§3.2-3.5, Alg. 1 at PAPER.md:436-481).  The hot operators run on the GPU (P2G, implicit
// solves, G2P, Pi, I, T); the once-per-frame receiver-set construction (boundary grid selection,
// overlap arbitration, eligibility) is host logic over node flags read back from the device.
// Readings of the paper: DESIGN.md R10-R16.
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

#include <map>

#include "dist.cuh"
#include "transmit.cuh"

struct osmpm_coupler {
    osmpm_subdomain* coarse = nullptr;
    osmpm_subdomain* fine = nullptr;
    osmpm_schwarz_settings set{};
    virtual ~osmpm_coupler() {}
    virtual osmpm_status prepare() = 0;
    virtual osmpm_status substep(int m, osmpm_solve_stats* st) = 0;
    virtual osmpm_status step(osmpm_schwarz_report* rep) = 0;
};

namespace osmpm {

// v = (1 - alpha) a + alpha b  (T_m, Eq. temporal_interp)
__global__ void k_lerp(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double alpha,
                       double* __restrict__ out)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (1.0 - alpha) * a[i] + alpha * b[i];
}

// ---------------------------------------------------------------------------------------------
// Host logic of one fine node box (a whole fine subdomain, or one slab with its ghost planes; R21):
// Gamma_S candidates (active, m^∂ > tau_S; Eq. boundary_grid_set), the arbitration of nodes that
// coincide with a coarse Gamma_B node (Eq. overlap_donor: the larger raw nodal mass donates, ties -> B;
// R12) and the eligibility of fine receivers (every coarse stencil node with N > 0 active; R13).
// Boxes: node (l0,l1,l2) of a box = dense node lo + l, box-local index (l0*n1 + l1)*n2 + l2.
// Out: dropB[I] |= 1 for coarse Gamma_B nodes a fine node takes over (B donates); cand[g] = owned?
// for the fine receivers (dense index g), owned = box-local index < nown.
// ---------------------------------------------------------------------------------------------
struct HostBox {
    int d;
    double o[3], dx;
    int64_t gd[3], lo[3], nn[3];
    int64_t nodes() const { return nn[0] * nn[1] * (d == 3 ? nn[2] : 1); }
    // box-local index of dense node k (or -1)
    int64_t local(const int64_t* k) const
    {
        int64_t l[3] = {0, 0, 0};
        for (int a = 0; a < d; ++a) {
            l[a] = k[a] - lo[a];
            if (k[a] < 0 || k[a] >= gd[a] || l[a] < 0 || l[a] >= nn[a]) return -1;
        }
        return d == 3 ? (l[0] * nn[1] + l[1]) * nn[2] + l[2] : l[0] * nn[1] + l[1];
    }
    int64_t dense(int64_t i, int64_t* k) const
    {
        int64_t l[3] = {0, 0, 0};
        if (d == 3) {
            l[2] = i % nn[2];
            l[1] = (i / nn[2]) % nn[1];
            l[0] = i / (nn[2] * nn[1]);
        } else {
            l[1] = i % nn[1];
            l[0] = i / nn[1];
        }
        for (int a = 0; a < 3; ++a) k[a] = a < d ? lo[a] + l[a] : 0;
        for (int a = 0; a < d; ++a)
            if (k[a] >= gd[a]) return -1;
        return d == 3 ? (k[0] * gd[1] + k[1]) * gd[2] + k[2] : k[0] * gd[1] + k[1];
    }
};

static inline double bspline_host(double f, int o)
{
    if (o == 0) return 0.5 * (1.5 - f) * (1.5 - f);
    if (o == 1) return 0.75 - (f - 1.0) * (f - 1.0);
    return 0.5 * (f - 0.5) * (f - 0.5);
}

inline void fine_box_receivers(const HostBox& Bx, const double* mB, const uint8_t* hatB, const uint8_t* actB,
                               const HostBox& Sx, int64_t nown, const double* mS, const double* mbS,
                               const uint8_t* actS, double tauS, uint8_t* dropB, std::map<int64_t, char>& cand)
{
    const int D = Sx.d;
    const double tol = 1e-9 * std::min(Bx.dx, Sx.dx);
    for (int64_t i = 0; i < Sx.nodes(); ++i) {
        if (!(actS[i] && mbS[i] > tauS)) continue;
        int64_t k[3];
        const int64_t g = Sx.dense(i, k);
        if (g < 0) continue;
        const bool owned = i < nown;
        bool keep = true;
        int64_t kk[3] = {0, 0, 0};
        bool coincide = true;
        for (int a = 0; a < D; ++a) {
            const double x = Sx.o[a] + Sx.dx * (double)k[a];
            const double X = (x - Bx.o[a]) / Bx.dx;
            kk[a] = (int64_t)std::llround(X);
            if (std::fabs(X - (double)kk[a]) * Bx.dx > tol || kk[a] < 0 || kk[a] >= Bx.gd[a]) coincide = false;
        }
        if (coincide) {
            const int64_t I = Bx.local(kk);
            if (I >= 0 && hatB[I]) {
                if (mB[I] >= mS[i])
                    dropB[I] = 1;  // B donates: S receives
                else
                    keep = false;  // S donates: B receives
            }
        }
        if (!keep) continue;
        double f[3];
        int64_t base[3] = {0, 0, 0};
        for (int a = 0; a < D; ++a) {
            const double x = Sx.o[a] + Sx.dx * (double)k[a];
            const double X = (x - Bx.o[a]) / Bx.dx;
            base[a] = (int64_t)std::floor(X - 0.5);
            f[a] = X - (double)base[a];
        }
        bool ok = true;
        for (int o0 = 0; o0 < 3 && ok; ++o0)
            for (int o1 = 0; o1 < 3 && ok; ++o1)
                for (int o2 = 0; o2 < (D == 3 ? 3 : 1) && ok; ++o2) {
                    const int off[3] = {o0, o1, o2};
                    double w = 1.0;
                    for (int a = 0; a < D; ++a) w *= bspline_host(f[a], off[a]);
                    if (!(w > 0.0)) continue;
                    int64_t kc[3] = {0, 0, 0};
                    for (int a = 0; a < D; ++a) kc[a] = base[a] + off[a];
                    const int64_t I = Bx.local(kc);
                    if (I < 0 || !actB[I]) ok = false;
                }
        if (!ok) continue;
        char& o = cand[g];  // a node seen by two local slabs: owned if either owns it
        o = (char)(o || owned);
    }
}

template <int D, typename R>
struct Coupler : public osmpm_coupler {
    Sub<D, R>* B = nullptr;   // coarse subdomain: never decomposed (replicated on every rank)
    Sub<D, R>* Ss = nullptr;  // fine subdomain, whole ...
    Dist<D, R>* Sd = nullptr; // ... or slab-decomposed (over this rank's local slabs and the ranks)
    std::vector<int64_t> recvB, recvS;           // receivers (dense node indices, ascending); recvS: this
    std::vector<char> ownS;                      // rank's slab boxes (owned + ghost planes), ownS: owned
    DBuf<int64_t> dB, dS;
    DBuf<uint8_t> maskB, maskS, flagsB;
    DBuf<double> vGB, vGBnew, vSn, vSnp1, vSprev, vbc, num, red2;
    bool prepared = false;
    double eps_tol = 0.0;
    cudaStream_t st() const { return B->st(); }
    SlabGroup<D, R> FG() { return Sd ? Sd->group() : Ss->self_group(); }
    bool multi() { return Sd && Sd->gc && Sd->gc->multi(); }
    GridGeo fine_geo() const { return Sd ? geo_of(Sd) : geo_of(Ss); }
    const int64_t* fine_gdims() const { return Sd ? Sd->gdims : Ss->gdims; }
    double fine_median_mass() { return FG().s[0]->median_mass; }
    double fine_total_mass() const { return Sd ? Sd->total_mass : Ss->total_mass; }
    double fine_dx() const { return Sd ? Sd->dx : Ss->dx; }
    const double* fine_origin() const { return Sd ? Sd->origin : Ss->origin; }

    // ------------------------------------------------------------------------------------------
    // host helpers
    // ------------------------------------------------------------------------------------------
    template <typename T>
    static osmpm_status d2h(std::vector<T>& h, const T* d, size_t n, cudaStream_t s)
    {
        h.resize(n);
        if (n) OSMPM_CU(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
        return OSMPM_OK;
    }

    // box-local index of a dense node index (or -1 outside the box)
    static int64_t box_of(const Sub<D, R>* s, int64_t g)
    {
        const BoxDev& b = s->box;
        int64_t k[3] = {0, 0, 0};
        if (D == 3) {
            k[2] = g % s->gdims[2];
            k[1] = (g / s->gdims[2]) % s->gdims[1];
            k[0] = g / (s->gdims[2] * s->gdims[1]);
        } else {
            k[1] = g % s->gdims[1];
            k[0] = g / s->gdims[1];
        }
        int64_t l[3];
        for (int a = 0; a < 3; ++a) {
            l[a] = (a < D) ? k[a] - b.lo[a] : 0;
            if (a < D && (l[a] < 0 || l[a] >= b.nn[a])) return -1;
        }
        return (D == 3) ? (l[0] * b.nn[1] + l[1]) * b.nn[2] + l[2] : l[0] * b.nn[1] + l[1];
    }

    static int64_t dense_of_box(const Sub<D, R>* s, int64_t i, int64_t* k)
    {
        const BoxDev& b = s->box;
        int64_t l[3] = {0, 0, 0};
        if (D == 3) {
            l[2] = i % b.nn[2];
            l[1] = (i / b.nn[2]) % b.nn[1];
            l[0] = i / ((int64_t)b.nn[2] * b.nn[1]);
        } else {
            l[1] = i % b.nn[1];
            l[0] = i / b.nn[1];
        }
        for (int a = 0; a < 3; ++a) k[a] = (a < D) ? b.lo[a] + l[a] : 0;
        for (int a = 0; a < D; ++a)
            if (k[a] >= s->gdims[a]) return -1;
        return (D == 3) ? (k[0] * s->gdims[1] + k[1]) * s->gdims[2] + k[2] : k[0] * s->gdims[1] + k[1];
    }

    static HostBox host_box(const Sub<D, R>* s)
    {
        HostBox h{};
        h.d = D;
        h.dx = s->dx;
        for (int a = 0; a < 3; ++a) {
            h.o[a] = s->origin[a];
            h.gd[a] = s->gdims[a];
            h.lo[a] = a < D ? s->box.lo[a] : 0;
            h.nn[a] = a < D ? s->box.nn[a] : 1;
        }
        return h;
    }

    // ------------------------------------------------------------------------------------------
    // Step 0: store, P2G both, Gamma, arbitration, receivers, v_GammaB^(0)
    //
    // A decomposed fine subdomain: every slab evaluates Gamma_S and the arbitration on ALL nodes of its
    // box (owned and ghost planes: their m, m^∂ and activity are consistent after the halo sums, so a
    // ghost node takes exactly its owner's decision, and this rank's Dirichlet data cover its ghosts);
    // the coarse nodes a fine donor takes over are OR-ed over the ranks (all-reduce max) and the coarse
    // Gamma_B is rank 0's (broadcast; the replicated coarse subdomain runs deterministically).
    // ------------------------------------------------------------------------------------------
    osmpm_status prepare() override
    {
        SlabGroup<D, R> G = FG();
        OSMPM_TRY(fine->checkpoint());
        OSMPM_TRY(B->p2g());
        OSMPM_TRY(fine->p2g());
        OSMPM_TRY(B->boundary_mass());
        for (int i = 0; i < G.ns; ++i) OSMPM_TRY(G.s[i]->boundary_mass());
        OSMPM_TRY(halo_sum<D, R>(G, {{&Sub<D, R>::mb, 1}}));
        // Pi denominator of the step-0 fine grid (eligibility of coarse receivers, R13)
        const int64_t nnB = B->dense_nodes();
        OSMPM_TRY(num.need((size_t)nnB * (D + 1)));
        OSMPM_TRY(project_accumulate_group<D, R>(G, B, false, num.p));
        std::vector<double> mB, mbB, denB;
        std::vector<uint8_t> aB;
        OSMPM_TRY(d2h(mB, B->m.p, B->box.nnodes, st()));
        OSMPM_TRY(d2h(mbB, B->mb.p, B->box.nnodes, st()));
        OSMPM_TRY(d2h(aB, B->act.p, B->box.nnodes, st()));
        OSMPM_TRY(d2h(denB, num.p + nnB * D, nnB, st()));
        OSMPM_CU(cudaStreamSynchronize(st()));
        const double tauB = set.tau_gamma_rel * B->median_mass, tauS = set.tau_gamma_rel * fine_median_mass();
        // Gamma_B = {active I : m^b_I > tau} (Eq. boundary_grid_set), coarse box indices
        std::vector<uint8_t> hatB(B->box.nnodes, 0), dropB(B->box.nnodes, 0);
        for (int64_t i = 0; i < B->box.nnodes; ++i) hatB[i] = aB[i] && mbB[i] > tauB;
        if (multi()) {
            OSMPM_TRY(flagsB.need(std::max<int64_t>(B->box.nnodes, 1)));
            OSMPM_CU(cudaMemcpyAsync(flagsB.p, hatB.data(), B->box.nnodes, cudaMemcpyHostToDevice, st()));
            OSMPM_NCCL(ncclBroadcast(flagsB.p, flagsB.p, B->box.nnodes, ncclUint8, 0, Sd->gc->comm, st()));
            OSMPM_CU(cudaMemcpyAsync(hatB.data(), flagsB.p, B->box.nnodes, cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
        }
        // fine Gamma_S candidates on every local slab's whole box (dense index -> owned?)
        std::map<int64_t, char> candS;
        const HostBox Bx = host_box(B);
        for (int si = 0; si < G.ns; ++si) {
            Sub<D, R>* S = G.s[si];
            std::vector<double> mS, mbS;
            std::vector<uint8_t> aS;
            OSMPM_TRY(d2h(mS, S->m.p, S->box.nnodes, st()));
            OSMPM_TRY(d2h(mbS, S->mb.p, S->box.nnodes, st()));
            OSMPM_TRY(d2h(aS, S->act.p, S->box.nnodes, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            fine_box_receivers(Bx, mB.data(), hatB.data(), aB.data(), host_box(S), S->nown, mS.data(), mbS.data(),
                               aS.data(), tauS, dropB.data(), candS);
        }
        if (multi()) {
            OSMPM_CU(cudaMemcpyAsync(flagsB.p, dropB.data(), B->box.nnodes, cudaMemcpyHostToDevice, st()));
            OSMPM_NCCL(ncclAllReduce(flagsB.p, flagsB.p, B->box.nnodes, ncclUint8, ncclMax, Sd->gc->comm, st()));
            OSMPM_CU(cudaMemcpyAsync(dropB.data(), flagsB.p, B->box.nnodes, cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
        }
        recvS.clear();
        ownS.clear();
        for (auto& kv : candS) {
            recvS.push_back(kv.first);
            ownS.push_back(kv.second);
        }
        // coarse receivers: Gamma_B minus the nodes a fine donor took, with fine support (R13)
        recvB.clear();
        for (int64_t i = 0; i < B->box.nnodes; ++i) {
            if (!hatB[i] || dropB[i]) continue;
            int64_t k[3];
            const int64_t g = dense_of_box(B, i, k);
            if (g >= 0 && denB[g] > tauB) recvB.push_back(g);
        }
        std::sort(recvB.begin(), recvB.end());
        const int64_t nB = recvB.size(), nS = recvS.size();
        OSMPM_TRY(dB.need(std::max<int64_t>(nB, 1)));
        OSMPM_TRY(dS.need(std::max<int64_t>(nS, 1)));
        OSMPM_TRY(maskB.need(std::max<int64_t>(nB, 1)));
        OSMPM_TRY(maskS.need(std::max<int64_t>(nS, 1)));
        OSMPM_TRY(red2.need(4));
        for (DBuf<double>* bb : {&vGB, &vGBnew})
            OSMPM_TRY(bb->need(std::max<int64_t>(nB, 1) * D));
        for (DBuf<double>* bb : {&vSn, &vSnp1, &vSprev, &vbc})
            OSMPM_TRY(bb->need(std::max<int64_t>(nS, 1) * D));
        if (nB) OSMPM_CU(cudaMemcpyAsync(dB.p, recvB.data(), nB * sizeof(int64_t), cudaMemcpyHostToDevice, st()));
        if (nS) OSMPM_CU(cudaMemcpyAsync(dS.p, recvS.data(), nS * sizeof(int64_t), cudaMemcpyHostToDevice, st()));
        OSMPM_CU(cudaMemsetAsync(maskB.p, (1 << D) - 1, std::max<int64_t>(nB, 1), st()));
        OSMPM_CU(cudaMemsetAsync(maskS.p, (1 << D) - 1, std::max<int64_t>(nS, 1), st()));
        // v_GammaB^(0) = Pi(v_S^n) on the coarse receivers (R16)
        eps_tol = set.eps_tol >= 0 ? set.eps_tol : 1e-12 * fine_total_mass();
        if (nB) {
            OSMPM_TRY(project_out<D, R>(st(), B, nB, dB.p, num.p, num.p + nnB * D, eps_tol, vGB.p));
        }
        // v_GammaS^(0) = I(v_B^n) (R15: r_S at k = 0 compares I(v_B^(1)) with I(v_B^n))
        if (nS) {
            B->KC();
            k_interp<D><<<nblk_all(nS, 256), 256, 0, st()>>>(nS, dS.p, fine_geo(), B->box, B->vn.p, nullptr, 0.0,
                                                             vSprev.p, B->err.p);
            OSMPM_LAUNCH_CHECK();
        }
        // the coarse subdomain's Schwarz Dirichlet data for the first coarse solve
        OSMPM_TRY(B->set_dirlist(B->dir_cpl, nB, dB.p, maskB.p, vGB.p, OSMPM_DEVICE));
        OSMPM_CU(cudaStreamSynchronize(st()));
        prepared = true;
        return OSMPM_OK;
    }

    // endpoint interpolations for the current coarse solve (Eq. spatial_interp_n)
    osmpm_status endpoints()
    {
        const int64_t nS = recvS.size();
        if (!nS) return OSMPM_OK;
        B->KC();
        k_interp<D><<<nblk_all(nS, 256), 256, 0, st()>>>(nS, dS.p, fine_geo(), B->box, B->vn.p, nullptr, 0.0, vSn.p,
                                                         B->err.p);
        B->KC();
        k_interp<D><<<nblk_all(nS, 256), 256, 0, st()>>>(nS, dS.p, fine_geo(), B->box, B->vnew.p, nullptr, 0.0,
                                                         vSnp1.p, B->err.p);
        OSMPM_LAUNCH_CHECK();
        return OSMPM_OK;
    }

    // one fine sub-step m of Alg. 1 lines 459-463 (+ P2G of the current state first, R14)
    osmpm_status substep(int m, osmpm_solve_stats* stats) override
    {
        if (!prepared) {
            set_error("schwarz_substep before schwarz_prepare");
            return OSMPM_E_STATE;
        }
        if (m < 1 || m > set.M) {
            set_error("sub-step m = %d outside [1, M = %d] (SPEC.md:330)", m, set.M);
            return OSMPM_E_INVALID_ARG;
        }
        if (m == 1) {
            if (!B->have_vnew) {
                set_error("schwarz_substep(1) needs the coarse subdomain's solve of this iteration");
                return OSMPM_E_STATE;
            }
            OSMPM_TRY(endpoints());
        }
        SlabGroup<D, R> G = FG();
        bool grid = true;
        for (int i = 0; i < G.ns; ++i) grid = grid && G.s[i]->have_grid;
        if (!grid) OSMPM_TRY(fine->p2g());
        const int64_t nS = recvS.size();
        const double alpha = (double)m / (double)set.M;  // Eq. temporal_interp
        if (nS) {
            B->KC();
            k_lerp<<<nblk_all(nS * D, 256), 256, 0, st()>>>(nS * D, vSn.p, vSnp1.p, alpha, vbc.p);
            OSMPM_LAUNCH_CHECK();
        }
        // every local slab gets this rank's receiver list (each keeps the nodes of its own box)
        for (int i = 0; i < G.ns; ++i)
            OSMPM_TRY(G.s[i]->set_dirlist(G.s[i]->dir_cpl, nS, dS.p, maskS.p, vbc.p, OSMPM_DEVICE));
        {
            const osmpm_status rc = fine->implicit_solve(&set.fine, stats);
            if (rc != OSMPM_OK) {
                prefix_error("fine solve, sub-step %d: ", m);
                return rc;
            }
        }
        if (m == set.M) {
            // v_GammaB^(k+1) = Pi(last sub-step's solved fine velocities) (R16)
            const int64_t nnB = B->dense_nodes();
            OSMPM_TRY(num.need((size_t)nnB * (D + 1)));
            OSMPM_TRY(project_accumulate_group<D, R>(G, B, true, num.p));
            const int64_t nB = recvB.size();
            if (nB) {
                OSMPM_TRY(project_out<D, R>(st(), B, nB, dB.p, num.p, num.p + nnB * D, eps_tol, vGBnew.p));
            }
        }
        return fine->g2p();
    }

    static void rel_parts(const std::vector<double>& nw, const std::vector<double>& old, const std::vector<char>* own,
                          double* num2, double* den2)
    {
        double a = 0.0, b = 0.0;
        for (size_t i = 0; i < nw.size(); ++i) {
            if (own && !(*own)[i / D]) continue;
            a += (nw[i] - old[i]) * (nw[i] - old[i]);
            b += nw[i] * nw[i];
        }
        *num2 = a;
        *den2 = b;
    }
    static double rel_of(double a, double b) { return b > 0.0 ? std::sqrt(a / b) : std::sqrt(a); }

    osmpm_status step(osmpm_schwarz_report* rep) override
    {
        osmpm_schwarz_report local{};
        osmpm_schwarz_report* RP = rep ? rep : &local;
        std::memset(RP, 0, sizeof(*RP));
        OSMPM_TRY(prepare());
        const int64_t nB = recvB.size(), nS = recvS.size();
        RP->n_recv_B = (int)nB;
        int64_t nS_own = 0;
        for (char o : ownS) nS_own += o ? 1 : 0;
        if (multi()) {
            double v = (double)nS_own;
            OSMPM_CU(cudaMemcpyAsync(red2.p, &v, sizeof(double), cudaMemcpyHostToDevice, st()));
            OSMPM_NCCL(ncclAllReduce(red2.p, red2.p, 1, ncclDouble, ncclSum, Sd->gc->comm, st()));
            OSMPM_CU(cudaMemcpyAsync(&v, red2.p, sizeof(double), cudaMemcpyDeviceToHost, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            nS_own = (int64_t)v;
        }
        RP->n_recv_S = (int)nS_own;
        const int n_iter = set.parity_fixed_k > 0 ? set.parity_fixed_k : set.k_max;
        std::vector<double> hGB, hGBnew, hSnp1, hSprev;
        for (int k = 0; k < n_iter; ++k) {
            // Step 1: coarse solve with Dirichlet Gamma-hat_B <- v_GammaB^(k) (Eq. implicit_solve_coarse),
            // restarting from the frozen step-0 coarse grid (R14)
            OSMPM_TRY(B->set_dirlist(B->dir_cpl, nB, dB.p, maskB.p, vGB.p, OSMPM_DEVICE));
            {
                const osmpm_status rc = B->implicit_solve(&set.coarse, nullptr);
                if (rc != OSMPM_OK) {
                    prefix_error("coarse solve, Schwarz iteration %d: ", k + 1);
                    return rc;
                }
            }
            // Step 2: restore the fine particles (Alg. 1) and sub-cycle
            OSMPM_TRY(fine->restore());
            OSMPM_TRY(fine->p2g());
            for (int m = 1; m <= set.M; ++m) {
                {
                    const osmpm_status rc = substep(m, nullptr);
                    if (rc != OSMPM_OK) {
                        prefix_error("Schwarz iteration %d, ", k + 1);
                        return rc;
                    }
                }
                RP->fine_substeps++;
            }
            // Step 3: interface residuals (Eqs. convergence_residuals / criterion); r_S over this rank's
            // owned receivers, summed over the ranks
            OSMPM_TRY(d2h(hGB, vGB.p, nB * D, st()));
            OSMPM_TRY(d2h(hGBnew, vGBnew.p, nB * D, st()));
            OSMPM_TRY(d2h(hSnp1, vSnp1.p, nS * D, st()));
            OSMPM_TRY(d2h(hSprev, vSprev.p, nS * D, st()));
            OSMPM_CU(cudaStreamSynchronize(st()));
            double bn, bd, sn, sd;
            rel_parts(hGBnew, hGB, nullptr, &bn, &bd);
            rel_parts(hSnp1, hSprev, &ownS, &sn, &sd);
            if (multi()) {
                double v[2] = {sn, sd};
                OSMPM_CU(cudaMemcpyAsync(red2.p, v, 2 * sizeof(double), cudaMemcpyHostToDevice, st()));
                OSMPM_NCCL(ncclAllReduce(red2.p, red2.p, 2, ncclDouble, ncclSum, Sd->gc->comm, st()));
                OSMPM_CU(cudaMemcpyAsync(v, red2.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st()));
                OSMPM_CU(cudaStreamSynchronize(st()));
                sn = v[0];
                sd = v[1];
            }
            const double rB = rel_of(bn, bd), rS = rel_of(sn, sd);
            if (k < 256) {
                RP->r_B[k] = rB;
                RP->r_S[k] = rS;
            }
            RP->iters = k + 1;
            std::swap(vGB.p, vGBnew.p);
            std::swap(vGB.cap, vGBnew.cap);
            if (nS) OSMPM_CU(cudaMemcpyAsync(vSprev.p, vSnp1.p, nS * D * sizeof(double), cudaMemcpyDeviceToDevice, st()));
            if (rB <= set.eps_conv && rS <= set.eps_conv) {
                RP->converged = 1;
                if (set.parity_fixed_k <= 0) break;
            }
        }
        // Step 4: post-convergence coarse G2P + advection with v_B^(k*+1)
        OSMPM_TRY(B->g2p());
        OSMPM_TRY(B->sync());
        OSMPM_TRY(fine->sync());
        B->dir_cpl.n = 0;
        {
            SlabGroup<D, R> G = FG();
            for (int i = 0; i < G.ns; ++i) G.s[i]->dir_cpl.n = 0;
        }
        prepared = false;
        if (!RP->converged && set.parity_fixed_k <= 0) {
            set_error("Schwarz iteration did not converge in k_max = %d iterations (r_B = %g, r_S = %g)", set.k_max,
                      RP->r_B[std::min(RP->iters, 256) - 1], RP->r_S[std::min(RP->iters, 256) - 1]);
            return OSMPM_E_SCHWARZ_NOT_CONVERGED;
        }
        return OSMPM_OK;
    }
};

inline osmpm_status coupler_create(osmpm_subdomain* coarse, osmpm_subdomain* fine, const osmpm_schwarz_settings* s,
                                   osmpm_coupler** out)
{
    osmpm_coupler* c = nullptr;
#define MK(DD, RR)                                                                                  \
    {                                                                                               \
        auto* q = new Coupler<DD, RR>();                                                            \
        q->B = static_cast<Sub<DD, RR>*>(coarse);                                                   \
        if (fine->decomposed)                                                                       \
            q->Sd = static_cast<Dist<DD, RR>*>(fine);                                               \
        else                                                                                        \
            q->Ss = static_cast<Sub<DD, RR>*>(fine);                                                \
        c = q;                                                                                      \
    }
    if (coarse->dim == 3 && coarse->prec == OSMPM_F64) MK(3, double)
    else if (coarse->dim == 2 && coarse->prec == OSMPM_F64) MK(2, double)
    else if (coarse->dim == 3) MK(3, float)
    else MK(2, float)
#undef MK
    c->coarse = coarse;
    c->fine = fine;
    // a decomposed fine subdomain over several ranks: the replicated coarse subdomain runs in the
    // deterministic scatter mode so that every rank's coarse solve is bitwise the same
    if (fine->decomposed && fine->ctx->gc.multi()) {
        if (coarse->dim == 3 && coarse->prec == OSMPM_F64) static_cast<Sub<3, double>*>(coarse)->det_force = true;
        else if (coarse->dim == 2 && coarse->prec == OSMPM_F64) static_cast<Sub<2, double>*>(coarse)->det_force = true;
        else if (coarse->dim == 3) static_cast<Sub<3, float>*>(coarse)->det_force = true;
        else static_cast<Sub<2, float>*>(coarse)->det_force = true;
    }
    c->set = *s;
    *out = c;
    return OSMPM_OK;
}
inline void coupler_destroy(osmpm_coupler* c) { delete c; }
inline osmpm_status coupler_prepare(osmpm_coupler* c) { return c->prepare(); }
inline osmpm_status coupler_substep(osmpm_coupler* c, int32_t m, osmpm_solve_stats* st) { return c->substep(m, st); }
inline osmpm_status coupler_step(osmpm_coupler* c, osmpm_schwarz_report* r) { return c->step(r); }

}  // namespace osmpm
