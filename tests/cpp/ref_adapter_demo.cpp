// ref_adapter_demo.cpp — the reference's own API usage, compiled against the
// reference headers, run twice: on the reference library (CPU) and through
// xscat_b200_ref_adapter.hpp on the B200.  Prints one PASS/FAIL line per
// check (acceptance_main.cpp style) and exits non-zero on any failure.
//   usage: ref_adapter_demo <data dir with materials/ spectra/ detector/>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <string>

#include "xscat/rng.hpp"
#include "xscat/synthetic.hpp"
#include "xscat_b200_ref_adapter.hpp"

using namespace xscat;
namespace fs = std::filesystem;

static int g_fail = 0;

static void check(bool ok, const char* what, const std::string& detail)
{
    std::printf("%s  %-52s %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
    if (!ok)
        ++g_fail;
}

int main(int argc, char** argv)
{
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <data dir>\n", argv[0]);
        return 2;
    }
    const fs::path data = argv[1];
    const Material w = load_material(data / "materials" / "water.mat");
    const Material al = load_material(data / "materials" / "aluminum.mat");
    const DetectorResponse resp = load_detector_response(data / "detector" / "gd2o2s_208um.csv");
    char buf[256];

    // acceptance criterion 2 inputs (acceptance_main.cpp:128-158)
    {
        const VoxelPhantom ph = make_cube_phantom(32, 0.2, 6.4, w, 1.0);
        const ScanGeometry g = make_circular_geometry(60.0, 40.0, 24, 24, 0.55, 1);
        const Spectrum spec = monochromatic_spectrum(100.0);
        SimConfig cfg;
        cfg.photons_total = 100000;
        cfg.splitting = 10;
        cfg.seed = 424242;
        const SimResult cpu = xscat::simulate_scatter_stats(ph, g, 0, spec, resp, cfg, 4);
        const SimResult gpu = xscat_b200::simulate_scatter_stats(ph, g, 0, spec, resp, cfg, 4);
        std::snprintf(buf, sizeof buf, "(ref %.9g, b200 %.9g; se %.3g / %.3g)", cpu.total, gpu.total,
                      cpu.total_std_error, gpu.total_std_error);
        check(std::abs(gpu.total - cpu.total) <= 1e-9 * cpu.total && gpu.histories == cpu.histories,
              "simulate_scatter_stats, criterion-2 inputs", buf);
    }
    // primary on a two-material rods phantom, polyenergetic
    {
        const VoxelPhantom ph = make_rods_phantom(48, 10.0 / 48, 4.5, 8.0, w, 1.0, 4, 0.6, 3.0, al, 2.699);
        const ScanGeometry g = make_circular_geometry(128.2, 86.2, 40, 32, 0.5, 6);
        Spectrum spec;
        for (int e = 20; e <= 148; e += 8)
            spec.bins.push_back({double(e), 1.0 / e});
        const DetectorImage cpu = xscat::simulate_primary(ph, g, 2, spec, resp, SimConfig{}, 4);
        const DetectorImage gpu = xscat_b200::simulate_primary(ph, g, 2, spec, resp, SimConfig{}, 4);
        double worst = 0.0;
        for (std::size_t i = 0; i < cpu.values.size(); ++i)
            worst = std::max(worst, std::abs(gpu.values[i] - cpu.values[i]) / cpu.values[i]);
        std::snprintf(buf, sizeof buf, "(max rel diff %.2e)", worst);
        check(worst <= 1e-12, "simulate_primary, rods + 17-bin spectrum", buf);

        SimConfig cfg;
        cfg.photons_total = 6000;
        cfg.splitting = 5;
        cfg.seed = 20240915;
        const ScanResult scan = xscat_b200::run_scan(ph, g, spec, resp, cfg, {0, 3, 5}, ScanQuantity::both, 4);
        bool same = scan.scatter.images.size() == 3 && scan.primary.images.size() == 3;
        const int idx[3] = {0, 3, 5};
        for (int i = 0; same && i < 3; ++i)
            same = scan.scatter.images[i].values ==
                       xscat_b200::simulate_scatter(ph, g, idx[i], spec, resp, cfg, 1).values &&
                   scan.primary.images[i].values ==
                       xscat_b200::simulate_primary(ph, g, idx[i], spec, resp, cfg, 1).values;
        check(same, "run_scan == per-angle calls (bitwise)", "");
        bool threw = false;
        try {
            xscat_b200::run_scan(ph, g, spec, resp, cfg, {}, ScanQuantity::both, 1);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("empty angle subset") != std::string::npos;
        }
        check(threw, "run_scan({}) throws runtime_error", "");
        threw = false;
        try {
            xscat_b200::run_scan(ph, g, spec, resp, cfg, {9}, ScanQuantity::both, 1);
        } catch (const std::out_of_range& e) {
            threw = std::string(e.what()).find("angle index") != std::string::npos;
        }
        check(threw, "run_scan({9}) throws out_of_range", "");
    }
    // post-processing (REF postprocess.cpp) bitwise
    {
        DetectorImage img(40, 33);
        for (std::size_t i = 0; i < img.values.size(); ++i)
            img.values[i] = std::sin(0.37 * i) + 0.01 * i;
        const SgFilterSpec f{7, 3};
        check(xscat_b200::sg_smooth(img, f).values == xscat::sg_smooth(img, f).values, "sg_smooth bitwise", "");
        check(xscat_b200::upsample_image(img, 80, 66).values == xscat::upsample_image(img, 80, 66).values,
              "upsample_image bitwise", "");
        check(xscat_b200::downsample_average(img, 20, 11).values ==
                  xscat::downsample_average(img, 20, 11).values,
              "downsample_average bitwise", "");
        ProjectionStack st = make_stack(40, 33, {0.0, 1.0, 2.0, 3.0});
        for (int k = 0; k < 4; ++k)
            for (std::size_t i = 0; i < img.values.size(); ++i)
                st.images[k].values[i] = img.values[i] * (k + 1);
        const std::vector<double> tgt = {0.0, 0.5, 2.25, 3.5, 6.0};
        const ProjectionStack a = xscat_b200::interpolate_angles(st, tgt), b = xscat::interpolate_angles(st, tgt);
        bool same = true;
        for (int k = 0; k < 5; ++k)
            same = same && a.images[k].values == b.images[k].values;
        check(same, "interpolate_angles bitwise", "");
        check(xscat_b200::sg_kernel(2, 2, 3) == xscat::sg_kernel(2, 2, 3), "sg_kernel bitwise", "");
        Spectrum sp;
        sp.bins = {{20.0, 0.001}, {40.0, 1.0}, {60.0, 2.0}, {80.0, 0.0}, {100.0, 0.5}};
        check(xscat_b200::apportion_photons(sp, 12345) == xscat::apportion_photons(sp, 12345),
              "apportion_photons", "");
    }
    { // correction-loop stages: REF correct_projections / intensity_to_attenuation
        const int nu = 37, nv = 29, n = 3;
        ProjectionStack a = make_stack(nu, nv, {0.0, 1.0, 2.0}), p = a, sc = a, inten = a;
        DetectorImage flat(nu, nv);
        for (int i = 0; i < n; ++i)
            for (std::size_t k = 0; k < a.images[i].values.size(); ++k) {
                const double x = 0.001 * (double)(k + 97 * i);
                a.images[i].values[k] = 1.0 + std::sin(x);
                p.images[i].values[k] = 0.5 + 0.4 * std::cos(3 * x);
                sc.images[i].values[k] = 0.1 * std::sin(7 * x); // some negative: clamped
                inten.images[i].values[k] = 0.2 + 0.1 * std::cos(x);
                flat.values[k] = 1.5;
            }
        std::size_t cr = 0, cg = 0;
        const ProjectionStack r = xscat::correct_projections(a, p, sc, &cr);
        const ProjectionStack g = xscat_b200::correct_projections(a, p, sc, &cg);
        double md = 0.0;
        for (int i = 0; i < n; ++i)
            for (std::size_t k = 0; k < r.images[i].values.size(); ++k)
                md = std::max(md, std::fabs(r.images[i].values[k] - g.images[i].values[k]));
        check(cr == cg && md <= 1e-14, "correct_projections (Eq. 8)", "max |diff| " + std::to_string(md));
        const ProjectionStack ar = xscat::intensity_to_attenuation(inten, flat);
        const ProjectionStack ag = xscat_b200::intensity_to_attenuation(inten, flat);
        md = 0.0;
        for (int i = 0; i < n; ++i)
            for (std::size_t k = 0; k < ar.images[i].values.size(); ++k)
                md = std::max(md, std::fabs(ar.images[i].values[k] - ag.images[i].values[k]));
        check(md <= 1e-14, "intensity_to_attenuation", "max |diff| " + std::to_string(md));
        p.images[1].values[5] = 0.0;
        bool threw = false;
        try {
            xscat_b200::correct_projections(a, p, sc);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("non-positive primary pixel") != std::string::npos;
        }
        check(threw, "correct_projections throws runtime_error", "");
    }
    { // FDK: REF fbp_reconstruct vs the device, bit for bit
        const int nu = 24, nv = 16, n = 48;
        ScanGeometry g = make_circular_geometry(60.0, 40.0, nu, nv, 0.5, n);
        ProjectionStack st = make_stack(nu, nv, g.angles);
        for (int i = 0; i < n; ++i)
            for (int iv = 0; iv < nv; ++iv)
                for (int iu = 0; iu < nu; ++iu)
                    st.images[i].values[(size_t)iv * nu + iu] =
                        std::exp(-((iu - 12.0) * (iu - 12.0) / 30.0 + (iv - 8.0) * (iv - 8.0) / 20.0)) *
                        (1.0 + 0.1 * std::sin((double)i));
        const std::array<int, 3> dims{12, 10, 8};
        const Vec3 vx = xscat::default_voxel_size(g, dims);
        const Volume a = xscat::fbp_reconstruct(st, g, dims, vx);
        const Volume b = xscat_b200::fbp_reconstruct(st, g, dims, xscat_b200::default_voxel_size(g, dims));
        check(a.values == b.values, "fbp_reconstruct bitwise", "");
    }
    { // segmentation (recon.cpp:159-322): REF vs the device, bit for bit
        Volume vol = make_volume(20, 21, 22, {0.1, 0.1, 0.1});
        CounterRng rng(29);
        for (auto& v : vol.values) {
            const double pick = rng.uniform();
            v = static_cast<float>(pick < 0.3 ? 10.0 + 3.0 * rng.uniform()
                                  : pick < 0.7 ? 25.0 + 4.0 * rng.uniform() : 45.0 + 5.0 * rng.uniform());
        }
        const auto ta = xscat::otsu_thresholds(vol, 3, 1024);
        const auto tb = xscat_b200::otsu_thresholds(vol, 3, 1024);
        check(ta == tb, "otsu_thresholds bitwise", "");
        const std::vector<ClassSpec> cmap{{0, 0.0}, {1, 1.0}, {2, 2.699}};
        const auto sa = xscat::segment_volume(vol, ta, cmap);
        const auto sb = xscat_b200::segment_volume(vol, tb, cmap);
        check(sa.labels == sb.labels, "segment_volume bitwise", "");
        const VoxelPhantom pa = xscat::to_density_phantom(vol, sa, {10, 7, 11}, {w, al});
        const VoxelPhantom pb = xscat_b200::to_density_phantom(vol, sb, {10, 7, 11}, {w, al});
        check(pa.material_id == pb.material_id && pa.density == pb.density && pa.voxel_size.x == pb.voxel_size.x &&
                  pa.origin.z == pb.origin.z,
              "to_density_phantom bitwise", "");
    }
    { // the whole loop (correction.cpp:137-266): REF's scatter-free fixed-point case
        const VoxelPhantom ph = make_cylinder_phantom(24, 0.3, 2.2, 5.0, w, 1.0);
        const ScanGeometry g = make_circular_geometry(60.0, 40.0, 24, 24, 0.5, 36);
        const Spectrum spec = monochromatic_spectrum(100.0);
        SimConfig sim;
        sim.photons_total = 2000;
        sim.splitting = 4;
        sim.seed = 99;
        std::vector<int> all(g.n_angles());
        for (int i = 0; i < g.n_angles(); ++i)
            all[i] = i;
        const ScanResult primary = xscat::run_scan(ph, g, spec, resp, sim, all, ScanQuantity::primary, 2);
        VoxelPhantom empty = make_empty_phantom(24, 24, 24, ph.voxel_size, ph.materials);
        const DetectorImage flat = xscat::simulate_primary(empty, g, 0, spec, resp, sim);
        CorrectionConfig cfg;
        cfg.n_iterations = 1;
        cfg.mc_nu = cfg.mc_nv = 12;
        cfg.recon_dims = {24, 24, 24};
        cfg.n_classes = 2;
        cfg.class_map = {ClassSpec{0, 0.0}, ClassSpec{1, 1.0}};
        cfg.sim = sim;
        const CorrectionResult a = xscat::run_iterative_correction(primary.primary, flat, g, spec, resp, cfg, {w});
        const CorrectionResult b = xscat_b200::run_iterative_correction(primary.primary, flat, g, spec, resp, cfg, {w});
        double md = 0.0, peak = 0.0;
        for (std::size_t i = 0; i < a.corrected_volume.values.size(); ++i) {
            md = std::max(md, (double)std::abs(a.corrected_volume.values[i] - b.corrected_volume.values[i]));
            peak = std::max(peak, (double)std::abs(a.corrected_volume.values[i]));
        }
        std::snprintf(buf, sizeof buf, "(ncc %.9f / %.9f, max |dvol| %.2g of %.3g)", a.reports[0].ncc_to_previous,
                      b.reports[0].ncc_to_previous, md, peak);
        check(std::abs(a.reports[0].ncc_to_previous - b.reports[0].ncc_to_previous) < 1e-9 && md <= 1e-5 * peak,
              "run_iterative_correction vs REF", buf);
    }
    std::printf("%s\n", g_fail ? "FAILED" : "all checks passed");
    return g_fail ? 1 : 0;
}
