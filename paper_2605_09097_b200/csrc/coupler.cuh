// coupler.cuh -- multiplicative Schwarz coupling of a coarse and a fine subdomain (§3.3-3.5,
// Alg. 1).  Placeholder entry points; the driver is implemented in coupler_impl (next milestone).
#pragma once
#include "transmit.cuh"

namespace osmpm {

inline osmpm_status coupler_create(osmpm_subdomain*, osmpm_subdomain*, const osmpm_schwarz_settings*, osmpm_coupler**)
{
    set_error("Schwarz coupler not built yet");
    return OSMPM_E_STATE;
}
inline void coupler_destroy(osmpm_coupler*) {}
inline osmpm_status coupler_prepare(osmpm_coupler*)
{
    set_error("Schwarz coupler not built yet");
    return OSMPM_E_STATE;
}
inline osmpm_status coupler_substep(osmpm_coupler*, int32_t, osmpm_solve_stats*)
{
    set_error("Schwarz coupler not built yet");
    return OSMPM_E_STATE;
}
inline osmpm_status coupler_step(osmpm_coupler*, osmpm_schwarz_report*)
{
    set_error("Schwarz coupler not built yet");
    return OSMPM_E_STATE;
}

}  // namespace osmpm
