// host_common.h — host-side pieces of libxscatgpu.so that need no GPU.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/xscat_gpu.h"
#include "xs_types.h"

namespace xsh {

// Status + message; thrown internally, converted to xs_status at the ABI.
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...);

// Sets the thread-local message (context-free calls) and returns code.
int set_error(int code, const std::string& msg);
const char* thread_error();

void validate_sim_config(const xs_sim_config& c);   // REF transport.cpp:26-40
void validate_spectrum(const xs_spectrum& s);       // REF spectrum.cpp:11-30
void validate_geometry(const xs_geometry& g);       // REF scan_geometry.cpp:9-26
std::vector<uint64_t> apportion(const xs_spectrum& s, uint64_t photons_total); // transport.cpp:42-64

struct Frame {
    double src[3], center[3], uaxis[3], normal[3];
};
Frame frame_of(const xs_geometry& g, int angle_idx); // REF scan_geometry.cpp:44-67

// Table1D::loglog / linear on the host (REF table.hpp:38-69).
double loglog(const xs_table& t, double x);
double linear(const xs_table& t, double x);

// Packs a material set into the fp64 table buffer; returns descriptors.
void pack_materials(const xs_material* mats, int n, std::vector<double>& buf,
                    xsd::MatDesc* out);
xsd::TabDesc pack_table(const xs_table& t, std::vector<double>& buf);

std::vector<double> sg_kernel(int left, int right, int polyorder); // postprocess.cpp:28-102
void validate_sg(int window, int polyorder);

// Scatter statistics finalize (transport.cpp:289-322) from the non-image words
// of an accumulator.  bins/ledger point at the accumulator's sections.
void finalize_stats(const xs_spectrum& spec, const std::vector<uint64_t>& counts,
                    uint64_t hist_begin, uint64_t hist_end, const uint64_t* bins,
                    const uint64_t* ledger, const xs_accum_units& units, xs_scatter_result* out);

} // namespace xsh
