// ref_cli_integration.cpp — INTEGRATION EXAMPLE, not part of the product.
//
// Shows how the reference's own CLI (REF tools/main.cpp:83-180) is pointed at
// the B200 projector: REF's run configuration, input loaders and file formats
// (run_config.cpp, phantom.cpp XVOX1, detector_image.cpp XPRJ1, volume.cpp
// XVOL1) are REF's compiled objects, linked as a library; only the compute
// calls are re-qualified to xscat_b200:: (include/xscat_b200_ref_adapter.hpp).
// The command bodies therefore follow REF's cmd_simulate / cmd_reconstruct /
// cmd_correct closely by design.  No native file-format or INI handling is
// claimed here (SURVEY.md §8(f) rank 4 is NOT done).
//
//   xscat_b200_cli <config.ini> simulate [--what primary|scatter|both] [--angles a:b | i,j,...]
//   xscat_b200_cli <config.ini> reconstruct <stack.xprj> [--flat flat.xprj] <out.xvol> <dim>
//   xscat_b200_cli <config.ini> correct <raw.xprj> <flat.xprj>
//   xscat_b200_cli synth-phantom <cylinder|rods|head> <n> <voxel_cm> <materials_dir> <out.xvox>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "xscat/run_config.hpp"
#include "xscat/synthetic.hpp"
#include "xscat/volume.hpp"
#include "xscat_b200_ref_adapter.hpp"

using namespace xscat;
namespace fs = std::filesystem;

namespace {

constexpr int kExitValidation = 2;

RunConfig load_config(const fs::path& path)
{
    std::vector<std::string> errors;
    RunConfig cfg = build_run_config(parse_ini(path), path.parent_path(), errors);
    validate_run_config(cfg, errors);
    if (!errors.empty()) {
        for (const auto& e : errors)
            std::cerr << "config error: " << e << "\n";
        std::exit(kExitValidation);
    }
    return cfg;
}

// REF tools/main.cpp parse_angle_list semantics: "a:b" (half-open) or a list
std::vector<int> angle_list(const std::string& text, int n_angles, bool given)
{
    std::vector<int> out;
    if (!given) {
        for (int i = 0; i < n_angles; ++i)
            out.push_back(i);
        return out;
    }
    if (const auto colon = text.find(':'); colon != std::string::npos) {
        const int a = std::stoi(text.substr(0, colon)), b = std::stoi(text.substr(colon + 1));
        for (int i = a; i < b; ++i)
            out.push_back(i);
        return out;
    }
    std::string item;
    std::istringstream in(text);
    while (std::getline(in, item, ','))
        if (!item.empty())
            out.push_back(std::stoi(item));
    return out;
}

int simulate(const fs::path& ini, int argc, char** argv)
{
    std::string what = "both", angles;
    bool angles_given = false;
    for (int i = 0; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        if (k == "--what")
            what = argv[i + 1];
        else if (k == "--angles") {
            angles = argv[i + 1];
            angles_given = true;
        } else {
            std::cerr << "unknown option " << k << "\n";
            return kExitValidation;
        }
    }
    RunConfig cfg = load_config(ini);
    LoadedInputs in = load_inputs(cfg);
    std::printf("effective seed: %llu\n", static_cast<unsigned long long>(cfg.sim.seed));
    ScanQuantity q = ScanQuantity::both;
    if (what == "primary")
        q = ScanQuantity::primary;
    else if (what == "scatter")
        q = ScanQuantity::scatter;
    else if (what != "both") {
        std::cerr << "--what must be primary|scatter|both\n";
        return kExitValidation;
    }
    const std::vector<int> subset = angle_list(angles, in.geometry.n_angles(), angles_given);
    if (subset.empty()) {
        std::cerr << "usage error: empty angle list\n";
        return kExitValidation;
    }
    for (int idx : subset)
        if (idx < 0 || idx >= in.geometry.n_angles()) {
            std::cerr << "angle index " << idx << " out of range\n";
            return kExitValidation;
        }
    fs::create_directories(cfg.output_dir);
    const ScanResult result =
        xscat_b200::run_scan(in.phantom, in.geometry, in.spectrum, in.response, cfg.sim, subset, q, cfg.threads);
    if (q != ScanQuantity::scatter)
        save_stack(result.primary, cfg.output_dir / "primary.xprj");
    if (q != ScanQuantity::primary)
        save_stack(result.scatter, cfg.output_dir / "scatter.xprj");
    std::ofstream timing(cfg.output_dir / "timing.csv");
    timing << "angle_idx,seconds\n";
    double total = 0.0;
    for (std::size_t i = 0; i < subset.size(); ++i) {
        timing << subset[i] << "," << result.seconds_per_angle[i] << "\n";
        total += result.seconds_per_angle[i];
    }
    timing << "total," << total << "\n";
    std::printf("simulated %zu angles in %.2f s (%.3f s/projection)\n", subset.size(), total,
                total / subset.size());
    return 0;
}

int reconstruct(const fs::path& ini, int argc, char** argv)
{
    std::vector<std::string> pos;
    std::string flat;
    for (int i = 0; i < argc; ++i) {
        if (std::string(argv[i]) == "--flat" && i + 1 < argc)
            flat = argv[++i];
        else
            pos.push_back(argv[i]);
    }
    if (pos.size() != 3) {
        std::cerr << "usage: reconstruct <stack.xprj> [--flat flat.xprj] <out.xvol> <dim>\n";
        return kExitValidation;
    }
    RunConfig cfg = load_config(ini);
    LoadedInputs in = load_inputs(cfg);
    ProjectionStack stack = load_stack(pos[0], in.geometry.angles);
    if (!flat.empty())
        stack = xscat_b200::intensity_to_attenuation(stack, load_stack(flat).images.at(0));
    const int dim = std::stoi(pos[2]);
    const std::array<int, 3> dims{dim, dim, dim};
    const Volume vol = xscat_b200::fbp_reconstruct(stack, in.geometry, dims,
                                                   xscat_b200::default_voxel_size(in.geometry, dims),
                                                   RampWindow::hann, cfg.threads);
    save_volume(vol, pos[1]);
    std::printf("wrote %s (%dx%dx%d)\n", pos[1].c_str(), dim, dim, dim);
    return 0;
}

int correct(const fs::path& ini, int argc, char** argv)
{
    if (argc != 2) {
        std::cerr << "usage: correct <raw.xprj> <flat.xprj>\n";
        return kExitValidation;
    }
    RunConfig cfg = load_config(ini);
    LoadedInputs in = load_inputs(cfg);
    std::printf("effective seed: %llu\n", static_cast<unsigned long long>(cfg.correction.sim.seed));
    const ProjectionStack raw = load_stack(argv[0], in.geometry.angles);
    const ProjectionStack flat = load_stack(argv[1]);
    fs::create_directories(cfg.output_dir);
    const CorrectionResult result = xscat_b200::run_iterative_correction(
        raw, flat.images.at(0), in.geometry, in.spectrum, in.response, cfg.correction, in.materials);
    save_volume(result.corrected_volume, cfg.output_dir / "corrected.xvol");
    save_stack(result.corrected_stack, cfg.output_dir / "corrected.xprj");
    write_reports(result.reports, cfg.output_dir / "reports.txt");
    write_summary_csv(result.reports, cfg.correction.sim, cfg.output_dir / "summary.csv");
    std::printf("corrected %d iterations in %.2f s\n", static_cast<int>(result.reports.size()),
                result.reports.empty() ? 0.0 : result.reports.back().seconds_total);
    return 0;
}

// Synthetic phantoms (REF synthetic.cpp) written as XVOX1, to drive the CLI.
int synth_phantom(int argc, char** argv)
{
    if (argc != 5) {
        std::cerr << "usage: synth-phantom <cylinder|rods|head> <n> <voxel_cm> <materials_dir> <out.xvox>\n";
        return kExitValidation;
    }
    const std::string kind = argv[0];
    const int n = std::stoi(argv[1]);
    const double vx = std::stod(argv[2]);
    const fs::path mats = argv[3];
    VoxelPhantom ph;
    if (kind == "cylinder")
        ph = make_cylinder_phantom(n, vx, 0.4 * n * vx, 0.8 * n * vx, load_material(mats / "water.mat"), 1.0);
    else if (kind == "rods")
        ph = make_rods_phantom(n, vx, 0.45 * n * vx, 0.8 * n * vx, load_material(mats / "water.mat"), 1.0, 4,
                               0.06 * n * vx, 0.3 * n * vx, load_material(mats / "aluminum.mat"), 2.699);
    else if (kind == "head")
        ph = make_cylinder_head_phantom(n, vx, load_material(mats / "aluminum.mat"), 2.699,
                                        load_material(mats / "iron.mat"), 7.874);
    else {
        std::cerr << "unknown phantom kind " << kind << "\n";
        return kExitValidation;
    }
    save_phantom(ph, argv[4]);
    std::printf("wrote %s (%d^3)\n", argv[4], n);
    return 0;
}

} // namespace

int main(int argc, char** argv)
{
    try {
        if (argc >= 2 && std::string(argv[1]) == "synth-phantom")
            return synth_phantom(argc - 2, argv + 2);
        if (argc < 3) {
            std::cerr << "usage: " << argv[0] << " <config.ini> simulate|reconstruct|correct ...\n";
            return kExitValidation;
        }
        const fs::path ini = argv[1];
        const std::string cmd = argv[2];
        if (cmd == "simulate")
            return simulate(ini, argc - 3, argv + 3);
        if (cmd == "reconstruct")
            return reconstruct(ini, argc - 3, argv + 3);
        if (cmd == "correct")
            return correct(ini, argc - 3, argv + 3);
        std::cerr << "unknown command " << cmd << "\n";
        return kExitValidation;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
