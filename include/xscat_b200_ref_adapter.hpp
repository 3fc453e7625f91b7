// xscat_b200_ref_adapter.hpp — drop-in replacement of the reference's
// projector API (include/xscat/transport.hpp:69-116 and
// include/xscat/postprocess.hpp:13-41) on the B200 library.
//
// Header-only C++17 over the C ABI of xscat_gpu.h.  It takes and returns the
// reference's own types, so a reference user switches a call site by
// qualifying it with xscat_b200:: (or with `using xscat_b200::...`), e.g. in
// REF src/correction.cpp:184-194:
//
//     ScanResult scatter_run = xscat_b200::run_scan(phantom, g_mc, spec, resp, cfg.sim,
//                                                   scatter_subset, ScanQuantity::scatter,
//                                                   cfg.workers);
//
// Errors are rethrown as the exception types the reference throws
// (xs_status -> std::runtime_error / out_of_range / invalid_argument /
// domain_error), with the reference's message text.  `workers` is accepted
// and ignored: results do not depend on it (or on the number of GPUs).
//
// Device selection: XSCAT_DEVICE (default 0).  One context per thread; the
// scene (phantom + response) is uploaded on every call, like the reference
// receives it on every call; Projector keeps it resident across calls.
// Several GPUs: XSCAT_DEVICES="0,1,2,3" (two or more entries) makes the
// projector calls and the correction loop run on an xs_group of those devices
// (photon batches for one projection, angle ranges for scans and the loop's
// scans; bit-identical results for any device list, REF PAPER.md:215).
#pragma once

#include <algorithm>
#include <array>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "xscat/correction.hpp"
#include "xscat/detector_image.hpp"
#include "xscat/postprocess.hpp"
#include "xscat/recon.hpp"
#include "xscat/transport.hpp"
#include "xscat_gpu.h"

namespace xscat_b200 {

inline void throw_status(int st, const xs_context* ctx)
{
    if (st == XS_OK)
        return;
    const std::string msg = xs_last_error(ctx);
    switch (st) {
    case XS_E_OUT_OF_RANGE:
        throw std::out_of_range(msg);
    case XS_E_INVALID_ARGUMENT:
        throw std::invalid_argument(msg);
    case XS_E_DOMAIN:
        throw std::domain_error(msg);
    default:
        throw std::runtime_error(msg);
    }
}

// ---------------------------------------------------------- type bridging
struct Packed {
    std::vector<xs_material> mats;
    xs_phantom ph{};
    xs_geometry g{};
    xs_spectrum s{};
    std::vector<double> se, sw;
    xs_response r{};
    xs_sim_config c{};
};

inline xs_table table_view(const xscat::Table1D& t)
{
    return xs_table{static_cast<int32_t>(t.size()), t.xs().data(), t.ys().data()};
}

inline void pack_phantom(Packed& p, const xscat::VoxelPhantom& ph)
{
    p.mats.resize(ph.materials.size());
    for (std::size_t i = 0; i < ph.materials.size(); ++i) {
        const xscat::Material& m = ph.materials[i];
        xs_material& x = p.mats[i];
        x.name = m.name.c_str();
        x.z_eff = m.z_eff;
        x.density_ref = m.density_ref;
        if (!m.has_tables()) {
            x.mu = x.sigma_incoh = x.sigma_coh = x.sigma_pe = x.s_factor = x.f_factor =
                xs_table{0, nullptr, nullptr};
            continue;
        }
        x.mu = table_view(m.mu);
        x.sigma_incoh = table_view(m.sigma_incoh);
        x.sigma_coh = table_view(m.sigma_coh);
        x.sigma_pe = table_view(m.sigma_pe);
        x.s_factor = table_view(m.s_factor);
        x.f_factor = table_view(m.f_factor);
    }
    for (int a = 0; a < 3; ++a)
        p.ph.dims[a] = ph.dims[a];
    p.ph.voxel_size[0] = ph.voxel_size.x;
    p.ph.voxel_size[1] = ph.voxel_size.y;
    p.ph.voxel_size[2] = ph.voxel_size.z;
    p.ph.origin[0] = ph.origin.x;
    p.ph.origin[1] = ph.origin.y;
    p.ph.origin[2] = ph.origin.z;
    p.ph.material_id = ph.material_id.data();
    p.ph.density = ph.density.data();
    p.ph.n_materials = static_cast<int32_t>(ph.materials.size());
    p.ph.materials = p.mats.data();
}

inline void pack_call(Packed& p, const xscat::ScanGeometry& g, const xscat::Spectrum& spec,
                      const xscat::SimConfig& cfg)
{
    p.g = xs_geometry{g.sdd, g.sod, g.nu, g.nv, g.pixel_pitch, g.n_angles(), g.angles.data()};
    p.se.clear();
    p.sw.clear();
    for (const auto& b : spec.bins) {
        p.se.push_back(b.energy_kev);
        p.sw.push_back(b.weight);
    }
    p.s = xs_spectrum{static_cast<int32_t>(spec.bins.size()), p.se.data(), p.sw.data()};
    p.c = xs_sim_config{cfg.photons_total, cfg.splitting,        cfg.roulette_survival,
                        cfg.roulette_wmin_rel, cfg.step_voxels,  cfg.max_interactions,
                        cfg.seed,              cfg.track_variance ? 1 : 0};
}

// ------------------------------------------------------------------ context
class Context {
public:
    explicit Context(int device = default_device())
    {
        throw_status(xs_ctx_create(device, &ctx_), nullptr);
    }
    ~Context() { xs_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    xs_context* get() const { return ctx_; }

    static int default_device()
    {
        const char* e = std::getenv("XSCAT_DEVICE");
        return e ? std::atoi(e) : 0;
    }

private:
    xs_context* ctx_ = nullptr;
};

inline Context& thread_context()
{
    thread_local Context ctx;
    return ctx;
}

inline void throw_group(int st, const xs_group* grp)
{
    if (st == XS_OK)
        return;
    const std::string msg = xs_group_last_error(grp);
    switch (st) {
    case XS_E_OUT_OF_RANGE:
        throw std::out_of_range(msg);
    case XS_E_INVALID_ARGUMENT:
        throw std::invalid_argument(msg);
    case XS_E_DOMAIN:
        throw std::domain_error(msg);
    default:
        throw std::runtime_error(msg);
    }
}

// A group of GPUs in this process (xs_group): one context per device.
class Group {
public:
    explicit Group(const std::vector<int>& devices)
    {
        std::vector<int32_t> d(devices.begin(), devices.end());
        throw_status(xs_group_create(d.data(), static_cast<int32_t>(d.size()), &grp_), nullptr);
    }
    ~Group() { xs_group_destroy(grp_); }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    xs_group* get() const { return grp_; }

    // XSCAT_DEVICES="0,1,...": the devices, or empty when unset / one entry
    static std::vector<int> devices_from_env()
    {
        std::vector<int> out;
        const char* e = std::getenv("XSCAT_DEVICES");
        if (!e)
            return out;
        for (const char* q = e; *q;) {
            out.push_back(std::atoi(q));
            while (*q && *q != ',')
                ++q;
            if (*q == ',')
                ++q;
        }
        if (out.size() < 2)
            out.clear();
        return out;
    }

private:
    xs_group* grp_ = nullptr;
};

// This thread's group when XSCAT_DEVICES names two or more devices, else null.
inline Group* thread_group()
{
    thread_local std::unique_ptr<Group> grp = [] {
        const std::vector<int> d = Group::devices_from_env();
        return d.empty() ? std::unique_ptr<Group>() : std::unique_ptr<Group>(new Group(d));
    }();
    return grp.get();
}

// A scene resident on the device (upload once, project many angles).
class Projector {
public:
    Projector(const xscat::VoxelPhantom& ph, const xscat::DetectorResponse& resp,
              Context& ctx = thread_context())
        : ctx_(ctx), grp_(thread_group())
    {
        Packed p;
        pack_phantom(p, ph);
        const xs_response r{table_view(resp.dqe), table_view(resp.deposit)};
        if (grp_) { // the scene on every device of the group (one upload, device-to-device copies)
            throw_group(xs_group_upload_response(grp_->get(), &r), grp_->get());
            throw_group(xs_group_upload_phantom(grp_->get(), &p.ph), grp_->get());
            return;
        }
        throw_status(xs_upload_phantom(ctx_.get(), &p.ph), ctx_.get());
        throw_status(xs_upload_response(ctx_.get(), &r), ctx_.get());
    }
    // Explicit group (overrides XSCAT_DEVICES).
    Projector(const xscat::VoxelPhantom& ph, const xscat::DetectorResponse& resp, Group& grp)
        : ctx_(thread_context()), grp_(&grp)
    {
        Packed p;
        pack_phantom(p, ph);
        const xs_response r{table_view(resp.dqe), table_view(resp.deposit)};
        throw_group(xs_group_upload_response(grp_->get(), &r), grp_->get());
        throw_group(xs_group_upload_phantom(grp_->get(), &p.ph), grp_->get());
    }

    // REF simulate_scatter_stats (transport.hpp:89-91)
    xscat::SimResult scatter_stats(const xscat::ScanGeometry& g, int angle_idx,
                                   const xscat::Spectrum& spec, const xscat::SimConfig& cfg) const
    {
        Packed p;
        pack_call(p, g, spec, cfg);
        xscat::SimResult out;
        out.image = xscat::DetectorImage(g.nu, g.nv);
        std::vector<double> var;
        if (cfg.track_variance)
            var.assign(out.image.values.size(), 0.0);
        xs_scatter_result r{};
        r.image = out.image.values.data();
        r.variance = cfg.track_variance ? var.data() : nullptr;
        if (grp_)
            throw_group(xs_group_simulate_scatter_stats(grp_->get(), &p.g, angle_idx, &p.s, &p.c, &r), grp_->get());
        else
            throw_status(xs_simulate_scatter_stats(ctx_.get(), &p.g, angle_idx, &p.s, &p.c, &r), ctx_.get());
        if (cfg.track_variance)
            out.image.variance = std::move(var);
        out.ledger.initial = r.ledger.initial;
        out.ledger.escaped = r.ledger.escaped;
        out.ledger.absorbed = r.ledger.absorbed;
        out.ledger.culled = r.ledger.culled;
        out.ledger.roulette_killed = r.ledger.roulette_killed;
        out.ledger.roulette_boost = r.ledger.roulette_boost;
        out.histories = r.histories;
        out.total = r.total;
        out.total_std_error = r.total_std_error;
        return out;
    }

    // REF simulate_primary (transport.hpp:100-102)
    xscat::DetectorImage primary(const xscat::ScanGeometry& g, int angle_idx,
                                 const xscat::Spectrum& spec, const xscat::SimConfig& cfg) const
    {
        Packed p;
        pack_call(p, g, spec, cfg);
        xscat::DetectorImage img(g.nu, g.nv);
        xs_context* c = grp_ ? xs_group_context(grp_->get(), 0) : ctx_.get();
        throw_status(xs_simulate_primary(c, &p.g, angle_idx, &p.s, &p.c, img.values.data()), c);
        return img;
    }

    // REF run_scan (transport.hpp:112-116)
    xscat::ScanResult scan(const xscat::ScanGeometry& g, const xscat::Spectrum& spec,
                           const xscat::SimConfig& cfg, const std::vector<int>& subset,
                           xscat::ScanQuantity what) const
    {
        Packed p;
        pack_call(p, g, spec, cfg);
        const std::size_t np = static_cast<std::size_t>(g.nu) * g.nv;
        const bool want_p = what != xscat::ScanQuantity::scatter;
        const bool want_s = what != xscat::ScanQuantity::primary;
        std::vector<double> prim(want_p ? np * subset.size() : 0), scat(want_s ? np * subset.size() : 0);
        std::vector<double> secs(subset.size());
        std::vector<int32_t> sub(subset.begin(), subset.end());
        const int q = what == xscat::ScanQuantity::primary ? 0 : (what == xscat::ScanQuantity::scatter ? 1 : 2);
        if (grp_)
            throw_group(xs_group_run_scan(grp_->get(), &p.g, &p.s, &p.c, sub.data(), static_cast<int32_t>(sub.size()),
                                          q, want_p ? prim.data() : nullptr, want_s ? scat.data() : nullptr,
                                          secs.data()),
                        grp_->get());
        else
            throw_status(xs_run_scan(ctx_.get(), &p.g, &p.s, &p.c, sub.data(), static_cast<int32_t>(sub.size()), q,
                                     want_p ? prim.data() : nullptr, want_s ? scat.data() : nullptr,
                                     secs.data()),
                         ctx_.get());
        std::vector<double> angles;
        for (int i : subset)
            angles.push_back(g.angles[i]);
        xscat::ScanResult out;
        if (want_p)
            out.primary = xscat::make_stack(g.nu, g.nv, angles);
        if (want_s)
            out.scatter = xscat::make_stack(g.nu, g.nv, angles);
        for (std::size_t i = 0; i < subset.size(); ++i) {
            if (want_p)
                std::copy(prim.begin() + i * np, prim.begin() + (i + 1) * np,
                          out.primary.images[i].values.begin());
            if (want_s)
                std::copy(scat.begin() + i * np, scat.begin() + (i + 1) * np,
                          out.scatter.images[i].values.begin());
        }
        out.seconds_per_angle = secs;
        return out;
    }

private:
    Context& ctx_;
    Group* grp_ = nullptr;
};

// ------------------------------------------- REF-signature free functions
inline xscat::SimResult simulate_scatter_stats(const xscat::VoxelPhantom& ph, const xscat::ScanGeometry& g,
                                               int angle_idx, const xscat::Spectrum& spec,
                                               const xscat::DetectorResponse& resp,
                                               const xscat::SimConfig& cfg, int /*workers*/ = 1)
{
    return Projector(ph, resp).scatter_stats(g, angle_idx, spec, cfg);
}

inline xscat::DetectorImage simulate_scatter(const xscat::VoxelPhantom& ph, const xscat::ScanGeometry& g,
                                             int angle_idx, const xscat::Spectrum& spec,
                                             const xscat::DetectorResponse& resp,
                                             const xscat::SimConfig& cfg, int workers = 1)
{
    return xscat_b200::simulate_scatter_stats(ph, g, angle_idx, spec, resp, cfg, workers).image;
}

inline xscat::DetectorImage simulate_primary(const xscat::VoxelPhantom& ph, const xscat::ScanGeometry& g,
                                             int angle_idx, const xscat::Spectrum& spec,
                                             const xscat::DetectorResponse& resp,
                                             const xscat::SimConfig& cfg, int /*workers*/ = 1)
{
    return Projector(ph, resp).primary(g, angle_idx, spec, cfg);
}

inline xscat::ScanResult run_scan(const xscat::VoxelPhantom& ph, const xscat::ScanGeometry& g,
                                  const xscat::Spectrum& spec, const xscat::DetectorResponse& resp,
                                  const xscat::SimConfig& cfg, const std::vector<int>& angle_subset,
                                  xscat::ScanQuantity what, int /*workers*/)
{
    return Projector(ph, resp).scan(g, spec, cfg, angle_subset, what);
}

inline std::vector<std::uint64_t> apportion_photons(const xscat::Spectrum& spec,
                                                    std::uint64_t photons_total)
{
    Packed p;
    pack_call(p, xscat::ScanGeometry{}, spec, xscat::SimConfig{});
    std::vector<std::uint64_t> out(spec.bins.size());
    throw_status(xs_apportion_photons(&p.s, photons_total, out.data()), nullptr);
    return out;
}

// ------------------------------------------------------ post-processing
inline std::vector<double> sg_kernel(int left, int right, int polyorder)
{
    std::vector<double> k(static_cast<std::size_t>(left + right + 1));
    throw_status(xs_sg_kernel(left, right, polyorder, k.data()), nullptr);
    return k;
}

inline xscat::SgFilterSpec default_sg_spec(int nu, int nv)
{
    int32_t w = 0, o = 0;
    xs_default_sg_spec(nu, nv, &w, &o);
    return xscat::SgFilterSpec{w, o};
}

inline xscat::DetectorImage sg_smooth(const xscat::DetectorImage& img, const xscat::SgFilterSpec& f)
{
    xscat::DetectorImage out(img.nu, img.nv);
    Context& c = thread_context();
    throw_status(xs_sg_smooth(c.get(), img.values.data(), out.values.data(), img.nu, img.nv, 1, f.window,
                              f.polyorder, 0),
                 c.get());
    return out;
}

inline xscat::ProjectionStack interpolate_angles(const xscat::ProjectionStack& stack,
                                                 const std::vector<double>& target_angles)
{
    const std::size_t np = static_cast<std::size_t>(stack.nu) * stack.nv;
    std::vector<double> in(np * stack.images.size()), out(np * target_angles.size());
    for (std::size_t i = 0; i < stack.images.size(); ++i)
        std::copy(stack.images[i].values.begin(), stack.images[i].values.end(), in.begin() + i * np);
    Context& c = thread_context();
    throw_status(xs_interpolate_angles(c.get(), in.data(), stack.angle_values.data(),
                                       static_cast<int32_t>(stack.angle_values.size()), out.data(),
                                       target_angles.data(), static_cast<int32_t>(target_angles.size()),
                                       stack.nu, stack.nv, 0),
                 c.get());
    xscat::ProjectionStack r = xscat::make_stack(stack.nu, stack.nv, target_angles);
    for (std::size_t i = 0; i < target_angles.size(); ++i)
        std::copy(out.begin() + i * np, out.begin() + (i + 1) * np, r.images[i].values.begin());
    return r;
}

inline xscat::DetectorImage upsample_image(const xscat::DetectorImage& img, int nu_out, int nv_out)
{
    xscat::DetectorImage out(nu_out, nv_out);
    Context& c = thread_context();
    throw_status(xs_upsample_image(c.get(), img.values.data(), img.nu, img.nv, 1, out.values.data(), nu_out,
                                   nv_out, 0),
                 c.get());
    return out;
}

inline xscat::DetectorImage downsample_average(const xscat::DetectorImage& img, int nu_out, int nv_out)
{
    xscat::DetectorImage out(nu_out, nv_out);
    Context& c = thread_context();
    throw_status(xs_downsample_average(c.get(), img.values.data(), img.nu, img.nv, 1, out.values.data(),
                                       nu_out, nv_out, 0),
                 c.get());
    return out;
}

// ------------------------------------------------ correction-loop stages
namespace detail {
inline std::vector<double> flatten(const xscat::ProjectionStack& s)
{
    const std::size_t np = static_cast<std::size_t>(s.nu) * s.nv;
    std::vector<double> v(np * s.images.size());
    for (std::size_t i = 0; i < s.images.size(); ++i)
        std::copy(s.images[i].values.begin(), s.images[i].values.end(), v.begin() + i * np);
    return v;
}

inline xscat::ProjectionStack unflatten(const std::vector<double>& v, int nu, int nv,
                                        const std::vector<double>& angles)
{
    xscat::ProjectionStack r = xscat::make_stack(nu, nv, angles);
    const std::size_t np = static_cast<std::size_t>(nu) * nv;
    for (std::size_t i = 0; i < r.images.size(); ++i)
        std::copy(v.begin() + i * np, v.begin() + (i + 1) * np, r.images[i].values.begin());
    return r;
}
} // namespace detail

// REF recon.hpp intensity_to_attenuation (recon.cpp:324-348)
inline xscat::ProjectionStack intensity_to_attenuation(const xscat::ProjectionStack& intensity,
                                                       const xscat::DetectorImage& flatfield)
{
    if (flatfield.nu != intensity.nu || flatfield.nv != intensity.nv)
        throw std::runtime_error("intensity_to_attenuation: flatfield dims mismatch");
    const std::vector<double> in = detail::flatten(intensity);
    std::vector<double> out(in.size());
    Context& c = thread_context();
    throw_status(xs_intensity_to_attenuation(c.get(), in.data(), flatfield.values.data(), intensity.nu,
                                             intensity.nv, intensity.n_angles(), out.data(), 0),
                 c.get());
    return detail::unflatten(out, intensity.nu, intensity.nv, intensity.angle_values);
}

// REF correction.hpp correct_projections (correction.cpp:58-86), Eq. 8
inline xscat::ProjectionStack correct_projections(const xscat::ProjectionStack& a, const xscat::ProjectionStack& primary,
                                                  const xscat::ProjectionStack& scatter,
                                                  std::size_t* clamped_count = nullptr)
{
    if (a.nu != primary.nu || a.nv != primary.nv || a.nu != scatter.nu || a.nv != scatter.nv ||
        a.n_angles() != primary.n_angles() || a.n_angles() != scatter.n_angles())
        throw std::runtime_error("correct_projections: stack dims mismatch");
    const std::vector<double> va = detail::flatten(a), vp = detail::flatten(primary), vs = detail::flatten(scatter);
    std::vector<double> out(va.size());
    uint64_t clamped = 0;
    Context& c = thread_context();
    throw_status(xs_correct_projections(c.get(), va.data(), vp.data(), vs.data(), a.nu, a.nv, a.n_angles(),
                                        out.data(), &clamped, 0),
                 c.get());
    if (clamped_count)
        *clamped_count = static_cast<std::size_t>(clamped);
    return detail::unflatten(out, a.nu, a.nv, a.angle_values);
}

// The loop's tail after the Monte Carlo runs (REF correction.cpp:199-246) in
// one device call: `scatter_run` = run_scan(..., scatter) on the angle subset
// (MC resolution), `primary_run` = the primary on every angle (MC
// resolution), `a` = the attenuation stack at full resolution.
inline xscat::ProjectionStack correction_tail(const xscat::ProjectionStack& scatter_run,
                                              const xscat::ProjectionStack& primary_run,
                                              const xscat::SgFilterSpec& sg, const xscat::ProjectionStack& a,
                                              double* mean_scatter_fraction = nullptr,
                                              std::size_t* clamped_count = nullptr)
{
    const std::vector<double> vs = detail::flatten(scatter_run), vp = detail::flatten(primary_run),
                              va = detail::flatten(a);
    std::vector<double> out(va.size());
    double frac = 0.0;
    uint64_t clamped = 0;
    Context& c = thread_context();
    throw_status(xs_correction_tail(c.get(), vs.data(), scatter_run.angle_values.data(), scatter_run.n_angles(),
                                    vp.data(), a.angle_values.data(), a.n_angles(), scatter_run.nu, scatter_run.nv,
                                    sg.window, sg.polyorder, va.data(), a.nu, a.nv, out.data(), &frac, &clamped, 0),
                 c.get());
    if (mean_scatter_fraction)
        *mean_scatter_fraction = frac;
    if (clamped_count)
        *clamped_count = static_cast<std::size_t>(clamped);
    return detail::unflatten(out, a.nu, a.nv, a.angle_values);
}

// REF recon.hpp default_voxel_size (recon.cpp:13-18)
inline xscat::Vec3 default_voxel_size(const xscat::ScanGeometry& g, const std::array<int, 3>& out_dims)
{
    const double fov = g.nu * g.pixel_pitch * g.sod / g.sdd;
    const double h = fov / std::max({out_dims[0], out_dims[1], out_dims[2]});
    return {h, h, h};
}

// REF recon.hpp fbp_reconstruct (recon.cpp:58-157) on the device; `workers`
// is accepted and ignored (the result does not depend on it).
inline xscat::Volume fbp_reconstruct(const xscat::ProjectionStack& stack, const xscat::ScanGeometry& g,
                                     const std::array<int, 3>& out_dims, const xscat::Vec3& voxel_size,
                                     xscat::RampWindow window = xscat::RampWindow::hann, int workers = 1)
{
    (void)workers;
    if (stack.images.empty())
        throw std::runtime_error("fbp: empty projection stack");
    const std::vector<double> v = detail::flatten(stack);
    xs_geometry xg{};
    xg.sdd = g.sdd;
    xg.sod = g.sod;
    xg.nu = g.nu;
    xg.nv = g.nv;
    xg.pixel_pitch = g.pixel_pitch;
    xg.angles = g.angles.data();
    xg.n_angles = static_cast<int32_t>(g.angles.size());
    const int32_t dims[3] = {out_dims[0], out_dims[1], out_dims[2]};
    const double vox[3] = {voxel_size.x, voxel_size.y, voxel_size.z};
    xscat::Volume vol = xscat::make_volume(out_dims[0], out_dims[1], out_dims[2], voxel_size);
    Context& c = thread_context();
    throw_status(xs_fbp_reconstruct(c.get(), v.data(), stack.angle_values.data(), stack.n_angles(), stack.nu,
                                    stack.nv, &xg, dims, vox, window == xscat::RampWindow::hann ? 1 : 0,
                                    vol.values.data(), 0),
                 c.get());
    return vol;
}

// ------------------------------------------------------------ segmentation
namespace detail {
inline std::vector<xs_class_spec> class_specs(const std::vector<xscat::ClassSpec>& m)
{
    std::vector<xs_class_spec> out;
    for (const auto& c : m)
        out.push_back(xs_class_spec{c.material_id, c.density});
    return out;
}

// REF material list (without vacuum) -> xs_material array with vacuum at 0
struct MaterialList {
    std::vector<xscat::Material> keep;
    std::vector<xs_material> xs;
    explicit MaterialList(const std::vector<xscat::Material>& mats)
    {
        keep.push_back(xscat::vacuum_material());
        for (const auto& m : mats)
            if (m.name != "vacuum")
                keep.push_back(m);
        xs.resize(keep.size());
        for (std::size_t i = 0; i < keep.size(); ++i) {
            const xscat::Material& m = keep[i];
            xs_material& x = xs[i];
            x.name = m.name.c_str();
            x.z_eff = m.z_eff;
            x.density_ref = m.density_ref;
            if (!m.has_tables()) {
                x.mu = x.sigma_incoh = x.sigma_coh = x.sigma_pe = x.s_factor = x.f_factor =
                    xs_table{0, nullptr, nullptr};
                continue;
            }
            x.mu = table_view(m.mu);
            x.sigma_incoh = table_view(m.sigma_incoh);
            x.sigma_coh = table_view(m.sigma_coh);
            x.sigma_pe = table_view(m.sigma_pe);
            x.s_factor = table_view(m.s_factor);
            x.f_factor = table_view(m.f_factor);
        }
    }
};
} // namespace detail

// REF recon.hpp otsu_thresholds (recon.cpp:159-240) on the device
inline std::vector<double> otsu_thresholds(const xscat::Volume& vol, int n_classes, int histogram_bins = 1024)
{
    Context& c = thread_context();
    const int32_t dims[3] = {vol.dims[0], vol.dims[1], vol.dims[2]};
    double thr[4] = {0, 0, 0, 0};
    throw_status(xs_otsu_thresholds(c.get(), vol.values.data(), dims, n_classes, histogram_bins, thr, 0), c.get());
    return std::vector<double>(thr, thr + std::max(0, n_classes - 1));
}

// REF recon.hpp segment_volume (recon.cpp:242-262)
inline xscat::SegmentationResult segment_volume(const xscat::Volume& vol, const std::vector<double>& thresholds,
                                                std::vector<xscat::ClassSpec> class_map)
{
    Context& c = thread_context();
    xscat::SegmentationResult seg;
    seg.labels.resize(vol.voxel_count());
    throw_status(xs_segment_volume(c.get(), vol.values.data(), vol.voxel_count(), thresholds.data(),
                                   static_cast<int32_t>(thresholds.size()), static_cast<int32_t>(class_map.size()),
                                   seg.labels.data(), 0),
                 c.get());
    seg.thresholds = thresholds;
    seg.class_map = std::move(class_map);
    return seg;
}

// REF recon.hpp to_density_phantom (recon.cpp:264-322)
inline xscat::VoxelPhantom to_density_phantom(const xscat::Volume& vol, const xscat::SegmentationResult& seg,
                                              const std::array<int, 3>& target_dims,
                                              std::vector<xscat::Material> materials)
{
    if (seg.labels.size() != vol.voxel_count())
        throw std::runtime_error("to_density_phantom: segmentation size mismatch");
    const xscat::Vec3 vs{vol.voxel_size.x * vol.dims[0] / target_dims[0],
                         vol.voxel_size.y * vol.dims[1] / target_dims[1],
                         vol.voxel_size.z * vol.dims[2] / target_dims[2]};
    xscat::VoxelPhantom ph = xscat::make_empty_phantom(target_dims[0], target_dims[1], target_dims[2], vs,
                                                       std::move(materials));
    detail::MaterialList ml(std::vector<xscat::Material>(ph.materials.begin() + 1, ph.materials.end()));
    const auto cls = detail::class_specs(seg.class_map);
    const int32_t src[3] = {vol.dims[0], vol.dims[1], vol.dims[2]};
    const int32_t tgt[3] = {target_dims[0], target_dims[1], target_dims[2]};
    Context& c = thread_context();
    throw_status(xs_to_density_phantom(c.get(), seg.labels.data(), src, cls.data(), static_cast<int32_t>(cls.size()),
                                       tgt, static_cast<int32_t>(ml.xs.size()), ml.xs.data(), ph.material_id.data(),
                                       ph.density.data(), 0),
                 c.get());
    return ph;
}

// REF correction.hpp run_iterative_correction (correction.cpp:137-266), every
// stage on the device; `workers` is ignored.  seconds_postprocess holds the
// fused post-processing + correction pass (seconds_correction is 0).
inline xscat::CorrectionResult run_iterative_correction(const xscat::ProjectionStack& raw_intensity,
                                                        const xscat::DetectorImage& flatfield,
                                                        const xscat::ScanGeometry& g, const xscat::Spectrum& spec,
                                                        const xscat::DetectorResponse& resp,
                                                        const xscat::CorrectionConfig& cfg,
                                                        const std::vector<xscat::Material>& materials)
{
    if (raw_intensity.n_angles() != g.n_angles())
        throw std::runtime_error("run_iterative_correction: stack angle count mismatch");
    Context& c = thread_context();
    Group* grp = thread_group(); // XSCAT_DEVICES: the loop's scans sharded over the group
    const xs_response r{table_view(resp.dqe), table_view(resp.deposit)};
    if (grp)
        throw_group(xs_group_upload_response(grp->get(), &r), grp->get());
    else
        throw_status(xs_upload_response(c.get(), &r), c.get());
    Packed p;
    pack_call(p, g, spec, cfg.sim);
    detail::MaterialList ml(materials);
    const auto cls = detail::class_specs(cfg.class_map);
    xs_correction_config cc;
    xs_correction_config_default(&cc);
    cc.n_iterations = cfg.n_iterations;
    cc.simulate_every_kth_angle = cfg.simulate_every_kth_angle;
    cc.mc_nu = cfg.mc_nu;
    cc.mc_nv = cfg.mc_nv;
    for (int a = 0; a < 3; ++a)
        cc.recon_dims[a] = cfg.recon_dims[a];
    cc.n_classes = cfg.n_classes;
    cc.class_map = cls.empty() ? nullptr : cls.data();
    cc.sim = p.c;
    cc.sg_window = cfg.sg.window;
    cc.sg_polyorder = cfg.sg.polyorder;
    cc.sg_auto_window = cfg.sg_auto_window ? 1 : 0;
    if (static_cast<int>(cfg.class_map.size()) != cfg.n_classes && cfg.n_classes >= 2 && cfg.n_classes <= 4)
        throw std::runtime_error("correction config: class_map must have n_classes entries");
    // the C call reads g.nu * g.nv * n_angles doubles of the stack and g.nu * g.nv
    // of the flat field: check the caller's dims first, with REF's messages
    // (REF recon.cpp:327-328; a stack that does not match the geometry fails
    // REF's Eq. 8 stage, correction.cpp:60-63 inside the stage wrapper :20-29)
    if (flatfield.nu != raw_intensity.nu || flatfield.nv != raw_intensity.nv ||
        flatfield.values.size() != static_cast<size_t>(flatfield.nu) * static_cast<size_t>(flatfield.nv))
        throw std::runtime_error("intensity_to_attenuation: flatfield dims mismatch");
    if (raw_intensity.n_angles() == g.n_angles() && (raw_intensity.nu != g.nu || raw_intensity.nv != g.nv))
        throw std::runtime_error("iteration 1, stage correction: correct_projections: stack dims mismatch");
    const std::vector<double> raw = detail::flatten(raw_intensity);
    xscat::CorrectionResult out;
    out.corrected_volume = xscat::make_volume(cfg.recon_dims[0], cfg.recon_dims[1], cfg.recon_dims[2],
                                              xscat::default_voxel_size(g, cfg.recon_dims));
    std::vector<double> stack(raw.size());
    std::vector<xs_iteration_report> reps(std::max(1, cfg.n_iterations));
    if (grp)
        throw_group(xs_group_run_iterative_correction(grp->get(), raw.data(), flatfield.values.data(), &p.g, &p.s,
                                                      &cc, static_cast<int32_t>(ml.xs.size()), ml.xs.data(),
                                                      out.corrected_volume.values.data(), stack.data(), reps.data(),
                                                      0),
                    grp->get());
    else
        throw_status(xs_run_iterative_correction(c.get(), raw.data(), flatfield.values.data(), &p.g, &p.s, &cc,
                                                 static_cast<int32_t>(ml.xs.size()), ml.xs.data(),
                                                 out.corrected_volume.values.data(), stack.data(), reps.data(), 0),
                     c.get());
    out.corrected_stack = detail::unflatten(stack, raw_intensity.nu, raw_intensity.nv, raw_intensity.angle_values);
    for (int i = 0; i < cfg.n_iterations; ++i) {
        const xs_iteration_report& x = reps[i];
        xscat::IterationReport rep;
        rep.iteration = x.iteration;
        rep.seconds_fbp = x.seconds_fbp;
        rep.seconds_segmentation = x.seconds_segmentation;
        rep.seconds_mc_scatter = x.seconds_mc_scatter;
        rep.seconds_mc_primary = x.seconds_mc_primary;
        rep.seconds_postprocess = x.seconds_postprocess;
        rep.seconds_correction = x.seconds_correction;
        rep.seconds_total = x.seconds_total;
        rep.mc_seconds_per_projection = x.mc_seconds_per_projection;
        rep.mean_scatter_fraction = x.mean_scatter_fraction;
        rep.ncc_to_previous = x.ncc_to_previous;
        rep.negative_scatter_clamped = x.negative_scatter_clamped;
        out.reports.push_back(rep);
    }
    return out;
}

} // namespace xscat_b200
