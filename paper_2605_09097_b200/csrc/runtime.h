// runtime.h -- host-side runtime of libosmpm: context, subdomain interface, error state.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "osmpm.h"

namespace osmpm {

void set_error(const char* fmt, ...);
void prefix_error(const char* fmt, ...);  // prepends context to the current message

#define OSMPM_CU(call)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            ::osmpm::set_error("CUDA error %s at %s:%d: %s", #call, __FILE__, __LINE__,             \
                               cudaGetErrorString(e_));                                             \
            return OSMPM_E_CUDA;                                                                    \
        }                                                                                           \
    } while (0)

#define OSMPM_TRY(...)                                                                              \
    do {                                                                                            \
        osmpm_status s_ = (__VA_ARGS__);                                                            \
        if (s_ != OSMPM_OK) return s_;                                                              \
    } while (0)

#define OSMPM_LAUNCH_CHECK()                                                                        \
    do {                                                                                            \
        cudaError_t e_ = cudaGetLastError();                                                        \
        if (e_ != cudaSuccess) {                                                                    \
            ::osmpm::set_error("kernel launch failed at %s:%d: %s", __FILE__, __LINE__,             \
                               cudaGetErrorString(e_));                                             \
            return OSMPM_E_CUDA;                                                                    \
        }                                                                                           \
    } while (0)

#define OSMPM_NCCL(call)                                                                            \
    do {                                                                                            \
        ncclResult_t r_ = (call);                                                                   \
        if (r_ != ncclSuccess) {                                                                    \
            ::osmpm::set_error("NCCL error %s at %s:%d: %s", #call, __FILE__, __LINE__,             \
                               ncclGetErrorString(r_));                                             \
            return OSMPM_E_NCCL;                                                                    \
        }                                                                                           \
    } while (0)

// Process group of the slab decomposition: one rank per GPU over NCCL (NVLink /
// NVSwitch).  Inside a rank the fine subdomain may additionally be split into `local_slabs`
// slabs on the same device, exchanging halos by device copies (the 1-GPU stand-in for the same
// decomposition: identical slab layout, halo and reduction logic, only the transport differs).
struct GroupComm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    int local_slabs = 1;
    bool multi() const { return comm != nullptr; }  // joined a communicator (of one or more ranks)
};

// CUDA-event timing of kernel families on the ctx stream
struct Profiler {
    bool on = false;
    struct Fam {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
        size_t used = 0;
    };
    std::map<std::string, Fam> fams;
    cudaEvent_t begin(const std::string& name, cudaStream_t s);
    void end(const std::string& name, cudaStream_t s);
    osmpm_status query(const std::string& name, int64_t* launches, double* ms);
    void reset();
    ~Profiler();
};

}  // namespace osmpm

struct osmpm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    osmpm::Profiler prof;
    int num_sms = 148;
    int64_t launches = 0;  // kernels launched through this ctx (bench gpu_launches)
    osmpm::GroupComm gc;
    // grow-only device scratch of the per-call operators (transmit): no cudaMalloc / cudaFree (an
    // implicit device synchronisation) inside a time step
    void* scratch[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t scratch_cap[6] = {0, 0, 0, 0, 0, 0};
    void* get_scratch(int k, size_t bytes)
    {
        if (scratch_cap[k] < bytes) {
            if (scratch[k]) cudaFree(scratch[k]);
            scratch[k] = nullptr;
            scratch_cap[k] = 0;
            if (cudaMalloc(&scratch[k], bytes + bytes / 8) != cudaSuccess) return nullptr;
            scratch_cap[k] = bytes + bytes / 8;
        }
        return scratch[k];
    }
};

struct osmpm_subdomain {
    osmpm_ctx* ctx = nullptr;
    int dim = 3;
    osmpm_precision prec = OSMPM_F64;
    bool decomposed = false;  // a Dist (slab-decomposed) subdomain
    virtual ~osmpm_subdomain() {}
    virtual osmpm_status set_gravity(const double* g) = 0;
    virtual osmpm_status set_dt(double dt) = 0;
    virtual osmpm_status set_particles(const double* x, const double* v, const double* F, const double* B,
                                       osmpm_memspace sp) = 0;
    virtual osmpm_status set_dirichlet(int64_t n, const int64_t* idx, const uint8_t* mask, const double* vel,
                                       osmpm_memspace sp) = 0;
    virtual osmpm_status p2g() = 0;
    virtual osmpm_status read_grid(double* m, double* p, double* v, double* fext, double* fsig, uint8_t* act,
                                   osmpm_memspace sp) = 0;
    virtual osmpm_status newton_gradient(const double* u, double* g, double* E, osmpm_memspace sp) = 0;
    virtual osmpm_status newton_hvp(const double* d, double* y, osmpm_memspace sp) = 0;
    virtual osmpm_status newton_diag(double* diag, osmpm_memspace sp) = 0;
    virtual osmpm_status implicit_solve(const osmpm_newton_settings* s, osmpm_solve_stats* st) = 0;
    virtual osmpm_status read_grid_velocity(double* v, osmpm_memspace sp) = 0;
    virtual osmpm_status set_grid_velocity(const double* v, osmpm_memspace sp) = 0;
    virtual osmpm_status g2p() = 0;
    virtual osmpm_status read_particles(double* x, double* v, double* F, double* B, osmpm_memspace sp) = 0;
    virtual osmpm_status info(int64_t* n, int64_t* lo, int64_t* dims) = 0;
    virtual osmpm_status sync() = 0;
    // a11: store / restore the whole particle state on the device
    virtual osmpm_status checkpoint() = 0;
    virtual osmpm_status restore() = 0;
};
