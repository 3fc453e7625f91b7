// xscat_b200 — the reference CLI's commands (`simulate`, `reconstruct`,
// `correct`, `phantom`, `metrics`, `inspect`) on the B200 library (SURVEY.md
// §8(f) rank 4; REF tools/main.cpp:83-310).
//
//   xscat_b200 simulate --config run.ini [--what primary|scatter|both]
//                       [--angles a:b | i,j,...] [--seed N] [--threads N]
//   xscat_b200 reconstruct --config run.ini --stack s.xprj [--flat f.xprj] --out v.xvol [--dim N]
//   xscat_b200 correct --config run.ini --raw raw.xprj --flat flat.xprj [--seed N]
//   xscat_b200 phantom --kind empty|cube|cylinder|rods|cylinder-head-like --out p.xvox [--dim N]
//                      [--voxel-cm X] [--radius-cm R] [--height-cm H] [--rods K] [--materials-dir D]
//   xscat_b200 metrics --a A [--b B] [--roi r,c,h,w,br,bc,bh,bw] [--slice N] [--out m.csv]
//                      [--profile r0,r1[,c0,c1]] [--profile-out p.csv]
//   xscat_b200 inspect --file f.xvox|f.xprj|f.xvol [--slice N] [--export out.pgm|out.csv]
//
// Native host code over the C ABI (include/xscat_gpu.h): the run configuration
// grammar and validation (REF run_config.cpp:84-247), the input loaders and
// file formats (csrc/files.cpp), the scan (xs_run_scan, or an xs_group when
// XSCAT_DEVICES lists several devices) and REF's outputs: primary.xprj,
// scatter.xprj and timing.csv in output_dir.  Messages and exit codes are
// REF's: 0 ok, 2 validation or usage error, 3 runtime error.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "xscat_gpu.h"

namespace fs = std::filesystem;

namespace {

constexpr int kExitValidation = 2;
constexpr int kExitRuntime = 3;

struct Failure { // a runtime error: "error: <msg>", exit 3
    std::string msg;
};

void check(int status, const char* (*msg)())
{
    if (status != XS_OK)
        throw Failure{msg()};
}

const char* lib_error() { return xs_last_error(nullptr); }

// the string without leading / trailing white space (the C locale's isspace set)
std::string strip(const std::string& s)
{
    static const char* const ws = " \t\n\v\f\r";
    const size_t first = s.find_first_not_of(ws);
    return first == std::string::npos ? std::string() : s.substr(first, s.find_last_not_of(ws) + 1 - first);
}

// "a, b,,c " -> {"a", "b", "c"}
std::vector<std::string> comma_list(const std::string& s)
{
    std::vector<std::string> items;
    for (size_t at = 0; at <= s.size();) {
        const size_t comma = std::min(s.find(',', at), s.size());
        const std::string item = strip(s.substr(at, comma - at));
        if (!item.empty())
            items.push_back(item);
        at = comma + 1;
    }
    return items;
}

// ------------------------------------------------------------ run config
// [section] blocks of key = value lines, '#' comments (REF run_config.cpp:84-113)
using Ini = std::map<std::string, std::map<std::string, std::string>>;

Ini read_ini(const fs::path& path)
{
    std::ifstream in(path);
    if (!in)
        throw Failure{"cannot open config file " + path.string()};
    Ini ini;
    std::string section, line;
    for (int no = 1; std::getline(in, line); ++no) {
        if (const size_t h = line.find('#'); h != std::string::npos)
            line.erase(h);
        line = strip(line);
        if (line.empty())
            continue;
        if (line.front() == '[') {
            if (line.back() != ']')
                throw Failure{path.string() + ":" + std::to_string(no) + ": malformed section header"};
            section = strip(line.substr(1, line.size() - 2));
            continue;
        }
        const size_t eq = line.find('=');
        if (eq == std::string::npos)
            throw Failure{path.string() + ":" + std::to_string(no) + ": expected key = value"};
        ini[section][strip(line.substr(0, eq))] = strip(line.substr(eq + 1));
    }
    return ini;
}

struct RunConfig { // REF run_config.hpp:16-45
    fs::path materials_dir, spectrum, response, phantom, output_dir = ".";
    std::vector<std::string> materials;
    double sdd = 0.0, sod = 0.0, pitch = 0.0;
    int nu = 0, nv = 0, n_angles = 0;
    xs_sim_config sim{};
    int n_iterations = 3, every_kth = 2, n_classes = 3;
    int mc_nu = 0, mc_nv = 0, recon_dim = 64, sg_window = 15, sg_polyorder = 3, sg_auto = 1;
    std::vector<std::string> class_map;
    int threads = 1;
};

// Keys, defaults and error texts of REF build_run_config (run_config.cpp:117-171).
class Reader {
public:
    Reader(const Ini& ini, std::vector<std::string>& errors) : ini_(ini), errors_(errors) {}
    std::string str(const std::string& sec, const std::string& key, const std::string& dflt, bool required)
    {
        if (auto s = ini_.find(sec); s != ini_.end())
            if (auto k = s->second.find(key); k != s->second.end())
                return strip(k->second);
        if (required)
            errors_.push_back("missing required key [" + sec + "] " + key);
        return dflt;
    }
    double num(const std::string& sec, const std::string& key, double dflt, bool required = false)
    {
        const std::string v = str(sec, key, "", required);
        if (v.empty())
            return dflt;
        try {
            size_t used = 0;
            const double x = std::stod(v, &used);
            if (used != v.size())
                throw std::invalid_argument(v);
            return x;
        } catch (...) {
            errors_.push_back("[" + sec + "] " + key + ": cannot parse number '" + v + "'");
            return dflt;
        }
    }
    long long integer(const std::string& sec, const std::string& key, long long dflt, bool required = false)
    {
        return static_cast<long long>(num(sec, key, static_cast<double>(dflt), required));
    }

private:
    const Ini& ini_;
    std::vector<std::string>& errors_;
};

RunConfig build_config(const Ini& ini, const fs::path& base, std::vector<std::string>& errors)
{
    Reader r(ini, errors);
    RunConfig c;
    auto at = [&](const std::string& p) -> fs::path {
        if (p.empty())
            return {};
        const fs::path q(p);
        return q.is_absolute() ? q : base / q;
    };
    c.materials_dir = at(r.str("paths", "materials_dir", "", true));
    c.materials = comma_list(r.str("paths", "materials", "", true));
    c.spectrum = at(r.str("paths", "spectrum", "", true));
    c.response = at(r.str("paths", "detector_response", "", true));
    c.phantom = at(r.str("paths", "phantom", "", true));
    c.output_dir = at(r.str("paths", "output_dir", ".", false));

    c.sdd = r.num("geometry", "sdd_cm", 0.0, true);
    c.sod = r.num("geometry", "sod_cm", 0.0, true);
    c.nu = static_cast<int>(r.integer("geometry", "det_nu", 0, true));
    c.nv = static_cast<int>(r.integer("geometry", "det_nv", 0, true));
    c.pitch = r.num("geometry", "pixel_pitch_cm", 0.0, true);
    c.n_angles = static_cast<int>(r.integer("geometry", "n_angles", 0, true));

    xs_sim_config_default(&c.sim);
    c.sim.photons_total = static_cast<uint64_t>(r.integer("sim", "photons_total", 10000));
    c.sim.splitting = static_cast<int>(r.integer("sim", "splitting", 1));
    c.sim.roulette_survival = r.num("sim", "roulette_survival", 0.5);
    c.sim.roulette_wmin_rel = r.num("sim", "roulette_wmin_rel", 1e-3);
    c.sim.step_voxels = static_cast<int>(r.integer("sim", "step_voxels", 1));
    c.sim.max_interactions = static_cast<int>(r.integer("sim", "max_interactions", 50));
    c.sim.seed = static_cast<uint64_t>(r.integer("sim", "seed", 0));

    c.n_iterations = static_cast<int>(r.integer("correction", "n_iterations", 3));
    c.every_kth = static_cast<int>(r.integer("correction", "simulate_every_kth_angle", 2));
    c.mc_nu = static_cast<int>(r.integer("correction", "mc_nu", 0));
    c.mc_nv = static_cast<int>(r.integer("correction", "mc_nv", 0));
    c.recon_dim = static_cast<int>(r.integer("correction", "recon_dim", 64));
    c.n_classes = static_cast<int>(r.integer("correction", "n_classes", 3));
    c.class_map = comma_list(r.str("correction", "class_map", "", false));
    c.sg_window = static_cast<int>(r.integer("correction", "sg_window", 15));
    c.sg_polyorder = static_cast<int>(r.integer("correction", "sg_polyorder", 3));
    c.sg_auto = r.integer("correction", "sg_auto_window", 1) != 0 ? 1 : 0;
    c.threads = static_cast<int>(r.integer("run", "threads", 1));
    return c;
}

// REF validate_run_config (run_config.cpp:173-230), in its order
void validate_config(const RunConfig& c, std::vector<std::string>& errors)
{
    auto file = [&](const fs::path& p, const std::string& what) {
        if (!p.empty() && !fs::exists(p))
            errors.push_back(what + " does not exist: " + p.string());
    };
    if (!c.materials_dir.empty() && !fs::is_directory(c.materials_dir))
        errors.push_back("materials_dir is not a directory: " + c.materials_dir.string());
    if (c.materials.empty())
        errors.push_back("no material files listed");
    for (const auto& m : c.materials)
        file(c.materials_dir / m, "material file");
    file(c.spectrum, "spectrum file");
    file(c.response, "detector response file");
    file(c.phantom, "phantom file");
    if (!(c.sod > 0.0) || !(c.sdd > c.sod))
        errors.push_back("geometry: require 0 < sod_cm < sdd_cm");
    if (c.nu <= 0 || c.nv <= 0)
        errors.push_back("geometry: det_nu/det_nv must be positive");
    if (!(c.pitch > 0.0))
        errors.push_back("geometry: pixel_pitch_cm must be positive");
    if (c.n_angles < 1)
        errors.push_back("geometry: n_angles must be >= 1");
    if (c.sim.photons_total < 1)
        errors.push_back("sim: photons_total must be >= 1");
    if (c.sim.splitting < 1)
        errors.push_back("sim: splitting must be >= 1");
    if (!(c.sim.roulette_survival > 0.0 && c.sim.roulette_survival <= 1.0))
        errors.push_back("sim: roulette_survival must lie in (0,1]");
    if (c.sim.step_voxels < 1)
        errors.push_back("sim: step_voxels must be >= 1");
    if (c.sim.max_interactions < 1)
        errors.push_back("sim: max_interactions must be >= 1");
    if (c.n_iterations < 1)
        errors.push_back("correction: n_iterations must be >= 1");
    if (c.every_kth < 1)
        errors.push_back("correction: simulate_every_kth_angle must be >= 1");
    if (c.n_classes < 2 || c.n_classes > 4)
        errors.push_back("correction: n_classes must be in [2,4]");
    if (!c.class_map.empty() && static_cast<int>(c.class_map.size()) != c.n_classes)
        errors.push_back("correction: class_map must list exactly n_classes entries");
    for (const auto& e : c.class_map)
        if (e.find(':') == std::string::npos)
            errors.push_back("correction: class_map entry '" + e + "' must be material:density");
    if (c.threads < 1)
        errors.push_back("run: threads must be >= 1");
}

// --------------------------------------------------------------- inputs
// REF load_inputs (run_config.cpp:232-266) through the library's loaders
struct Inputs {
    std::vector<xs_material_file*> files;
    std::vector<xs_material> materials; // [0] = vacuum
    xs_spectrum_file* spectrum = nullptr;
    xs_response_file* response = nullptr;
    xs_phantom_file* phantom_file = nullptr;
    xs_phantom phantom{};
    std::vector<double> angles;
    xs_geometry geometry{};
    std::vector<xs_class_spec> classes; // the resolved class map
    ~Inputs()
    {
        for (auto* f : files)
            xs_material_file_free(f);
        xs_spectrum_file_free(spectrum);
        xs_response_file_free(response);
        xs_phantom_file_free(phantom_file);
    }
};

void load_inputs(const RunConfig& c, Inputs& in)
{
    xs_material vacuum{};
    vacuum.name = "vacuum";
    in.materials.push_back(vacuum);
    for (const auto& m : c.materials) {
        xs_material_file* f = nullptr;
        check(xs_material_file_load((c.materials_dir / m).string().c_str(), &f), lib_error);
        in.files.push_back(f);
        in.materials.push_back(*xs_material_file_get(f));
    }
    check(xs_spectrum_file_load(c.spectrum.string().c_str(), &in.spectrum), lib_error);
    check(xs_response_file_load(c.response.string().c_str(), &in.response), lib_error);

    check(xs_phantom_file_read(c.phantom.string().c_str(), (uint32_t)in.materials.size(), &in.phantom_file),
          lib_error);
    xs_phantom& p = in.phantom;
    p = *xs_phantom_file_get(in.phantom_file);
    p.n_materials = (int32_t)in.materials.size();
    p.materials = in.materials.data();
    check(xs_validate_phantom(&p), lib_error); // REF load_phantom (phantom.cpp:159)

    // REF make_circular_geometry (scan_geometry.cpp:28-42)
    in.angles.resize(c.n_angles);
    for (int i = 0; i < c.n_angles; ++i)
        in.angles[i] = 2.0 * 3.14159265358979323846 * i / c.n_angles;
    in.geometry = xs_geometry{c.sdd, c.sod, c.nu, c.nv, c.pitch, c.n_angles, in.angles.data()};

    // the class map names loaded materials (REF resolves it on every command)
    for (const auto& e : c.class_map) {
        const std::string name = e.substr(0, e.find(':'));
        const double density = std::stod(e.substr(e.find(':') + 1));
        xs_class_spec cs{0, 0.0};
        if (name != "air" && name != "vacuum") {
            int id = -1;
            for (size_t i = 1; i < in.materials.size(); ++i)
                if (name == in.materials[i].name)
                    id = (int)i;
            if (id < 0)
                throw Failure{"class_map references unknown material '" + name + "'"};
            cs = xs_class_spec{id, density};
        }
        in.classes.push_back(cs);
    }
}

// ------------------------------------------------------------- commands
struct Flags {
    std::string config;
    std::optional<uint64_t> seed;
    std::optional<int> threads;
};

RunConfig config_or_exit(const Flags& f)
{
    const fs::path path = f.config;
    const Ini ini = read_ini(path);
    std::vector<std::string> errors;
    RunConfig c = build_config(ini, path.parent_path(), errors);
    if (f.seed)
        c.sim.seed = *f.seed;
    if (f.threads)
        c.threads = *f.threads;
    validate_config(c, errors);
    if (!errors.empty()) {
        std::cerr << "config validation failed (" << errors.size() << " problems):\n";
        for (const auto& e : errors)
            std::cerr << "  - " << e << "\n";
        std::exit(kExitValidation);
    }
    return c;
}

// "a:b" (half-open range) or a comma list; all angles when the flag is absent
std::vector<int> angle_subset(const std::string& text, int n, bool given)
{
    std::vector<int> out;
    if (!given) {
        for (int i = 0; i < n; ++i)
            out.push_back(i);
        return out;
    }
    if (const size_t colon = text.find(':'); colon != std::string::npos) {
        for (int i = std::stoi(text.substr(0, colon)), e = std::stoi(text.substr(colon + 1)); i < e; ++i)
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

std::vector<int32_t> devices_from_env()
{
    std::vector<int32_t> d;
    if (const char* e = std::getenv("XSCAT_DEVICES"))
        for (const auto& s : comma_list(e))
            d.push_back(std::stoi(s));
    return d;
}

int cmd_simulate(const Flags& flags, const std::string& what, const std::string& angles, bool angles_given)
{
    const RunConfig c = config_or_exit(flags);
    Inputs in;
    load_inputs(c, in);
    std::printf("effective seed: %llu\n", static_cast<unsigned long long>(c.sim.seed));
    int32_t q = 2; // ScanQuantity order: primary, scatter, both
    if (what == "primary")
        q = 0;
    else if (what == "scatter")
        q = 1;
    else if (what != "both") {
        std::cerr << "--what must be primary|scatter|both\n";
        return kExitValidation;
    }
    const std::vector<int> subset = angle_subset(angles, c.n_angles, angles_given);
    if (subset.empty()) {
        std::cerr << "usage error: empty angle list\n";
        return kExitValidation;
    }
    for (int a : subset)
        if (a < 0 || a >= c.n_angles) {
            std::cerr << "angle index " << a << " out of range\n";
            return kExitValidation;
        }
    fs::create_directories(c.output_dir);

    const size_t np = (size_t)c.nu * c.nv, n = subset.size();
    std::vector<double> prim(q != 1 ? n * np : 0), scat(q != 0 ? n * np : 0), secs(n);
    const std::vector<int32_t> sub(subset.begin(), subset.end());
    const std::vector<int32_t> devs = devices_from_env();
    if (devs.size() >= 2) { // one process, several devices (REF PAPER.md:215)
        xs_group* g = nullptr;
        check(xs_group_create(devs.data(), (int32_t)devs.size(), &g), lib_error);
        auto err = [g] { return std::string(xs_group_last_error(g)); };
        int st = xs_group_upload_phantom(g, &in.phantom);
        if (st == XS_OK)
            st = xs_group_upload_response(g, xs_response_file_get(in.response));
        if (st == XS_OK)
            st = xs_group_run_scan(g, &in.geometry, xs_spectrum_file_get(in.spectrum), &c.sim, sub.data(),
                                   (int32_t)n, q, prim.empty() ? nullptr : prim.data(),
                                   scat.empty() ? nullptr : scat.data(), secs.data());
        const std::string msg = st == XS_OK ? "" : err();
        xs_group_destroy(g);
        if (st != XS_OK)
            throw Failure{msg};
    } else {
        const char* dev = std::getenv("XSCAT_DEVICE");
        xs_context* ctx = nullptr;
        check(xs_ctx_create(dev ? std::atoi(dev) : 0, &ctx), lib_error);
        int st = xs_upload_phantom(ctx, &in.phantom);
        if (st == XS_OK)
            st = xs_upload_response(ctx, xs_response_file_get(in.response));
        if (st == XS_OK)
            st = xs_run_scan(ctx, &in.geometry, xs_spectrum_file_get(in.spectrum), &c.sim, sub.data(), (int32_t)n,
                             q, prim.empty() ? nullptr : prim.data(), scat.empty() ? nullptr : scat.data(),
                             secs.data());
        const std::string msg = st == XS_OK ? "" : xs_last_error(ctx);
        xs_ctx_destroy(ctx);
        if (st != XS_OK)
            throw Failure{msg};
    }
    if (q != 1)
        check(xs_stack_file_save((c.output_dir / "primary.xprj").string().c_str(), c.nu, c.nv, (int32_t)n,
                                 prim.data()),
              lib_error);
    if (q != 0)
        check(xs_stack_file_save((c.output_dir / "scatter.xprj").string().c_str(), c.nu, c.nv, (int32_t)n,
                                 scat.data()),
              lib_error);
    std::ofstream timing(c.output_dir / "timing.csv");
    timing << "angle_idx,seconds\n";
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) {
        timing << subset[i] << "," << secs[i] << "\n";
        total += secs[i];
    }
    timing << "total," << total << "\n";
    std::printf("simulated %zu angles in %.2f s (%.3f s/projection)\n", n, total, total / n);
    return 0;
}

// A projection stack file (REF load_stack): images widened to double;
// `angles` (may be empty) must have one entry per image.
struct Stack {
    int32_t nu = 0, nv = 0, n = 0;
    std::vector<double> images;
};

Stack load_stack(const std::string& path, const std::vector<double>& angles)
{
    Stack st;
    check(xs_stack_file_info(path.c_str(), &st.nu, &st.nv, &st.n), lib_error);
    if (!angles.empty() && (int)angles.size() != st.n)
        throw Failure{path + ": angle list size does not match file (" + std::to_string(angles.size()) + " vs " +
                      std::to_string(st.n) + ")"};
    st.images.resize((size_t)st.nu * st.nv * st.n);
    check(xs_stack_file_load(path.c_str(), st.images.data()), lib_error);
    return st;
}

// The context every device command runs on (XSCAT_DEVICE, default 0).
struct Device {
    xs_context* ctx = nullptr;
    Device()
    {
        const char* dev = std::getenv("XSCAT_DEVICE");
        check(xs_ctx_create(dev ? std::atoi(dev) : 0, &ctx), lib_error);
    }
    ~Device() { xs_ctx_destroy(ctx); }
    void ok(int st) const
    {
        if (st != XS_OK)
            throw Failure{xs_last_error(ctx)};
    }
};

// REF cmd_reconstruct (tools/main.cpp:132-150): FDK (Hann) of a stack, after
// the ln conversion against a flat field when one is given.
int cmd_reconstruct(const Flags& flags, const std::string& stack_path, const std::string& flat_path,
                    const std::string& out_path, int dim)
{
    const RunConfig c = config_or_exit(flags);
    Inputs in;
    load_inputs(c, in);
    Stack st = load_stack(stack_path, in.angles);
    Device d;
    if (!flat_path.empty()) {
        const Stack flat = load_stack(flat_path, {});
        if (flat.n < 1)
            throw Failure{"vector::_M_range_check: __n (which is 0) >= this->size() (which is 0)"};
        if (flat.nu != st.nu || flat.nv != st.nv)
            throw Failure{"intensity_to_attenuation: flatfield dims mismatch"};
        std::vector<double> att(st.images.size());
        d.ok(xs_intensity_to_attenuation(d.ctx, st.images.data(), flat.images.data(), st.nu, st.nv, st.n, att.data(), 0));
        st.images.swap(att);
    }
    const int32_t dims[3] = {dim, dim, dim};
    double voxel[3];
    xs_default_voxel_size(&in.geometry, dims, voxel);
    std::vector<float> vol((size_t)dim * dim * dim);
    d.ok(xs_fbp_reconstruct(d.ctx, st.images.data(), in.angles.data(), st.n, st.nu, st.nv, &in.geometry, dims, voxel,
                            1, vol.data(), 0));
    check(xs_volume_file_save(out_path.c_str(), dims, voxel, vol.data()), lib_error);
    std::printf("wrote %s (%dx%dx%d)\n", out_path.c_str(), dim, dim, dim);
    return 0;
}

// REF cmd_correct (tools/main.cpp:152-177): the iterative correction loop,
// then corrected.xvol, corrected.xprj, iterations.txt and summary.csv.
int cmd_correct(const Flags& flags, const std::string& raw_path, const std::string& flat_path)
{
    const RunConfig c = config_or_exit(flags);
    Inputs in;
    load_inputs(c, in);
    std::printf("effective seed: %llu\n", static_cast<unsigned long long>(c.sim.seed));
    const Stack raw = load_stack(raw_path, in.angles);
    const Stack flat = load_stack(flat_path, {});
    if (flat.n < 1)
        throw Failure{"vector::_M_range_check: __n (which is 0) >= this->size() (which is 0)"};
    fs::create_directories(c.output_dir);

    xs_correction_config cc;
    xs_correction_config_default(&cc);
    cc.n_iterations = c.n_iterations;
    cc.simulate_every_kth_angle = c.every_kth;
    cc.mc_nu = c.mc_nu;
    cc.mc_nv = c.mc_nv;
    cc.recon_dims[0] = cc.recon_dims[1] = cc.recon_dims[2] = c.recon_dim;
    cc.n_classes = c.n_classes;
    cc.class_map = in.classes.empty() ? nullptr : in.classes.data();
    cc.sim = c.sim;
    cc.sg_window = c.sg_window;
    cc.sg_polyorder = c.sg_polyorder;
    cc.sg_auto_window = c.sg_auto;
    // REF: flatfield dims against the raw stack (intensity_to_attenuation)
    if (flat.nu != raw.nu || flat.nv != raw.nv)
        throw Failure{"intensity_to_attenuation: flatfield dims mismatch"};
    if (raw.nu != c.nu || raw.nv != c.nv)
        throw Failure{"iteration 1, stage correction: correct_projections: stack dims mismatch"};

    const int n_it = std::max(c.n_iterations, 0);
    std::vector<xs_iteration_report> reports((size_t)std::max(n_it, 1));
    const int32_t dims[3] = {c.recon_dim, c.recon_dim, c.recon_dim};
    std::vector<float> vol((size_t)c.recon_dim * c.recon_dim * c.recon_dim);
    std::vector<double> stack(raw.images.size());
    Device d;
    d.ok(xs_upload_response(d.ctx, xs_response_file_get(in.response)));
    d.ok(xs_run_iterative_correction(d.ctx, raw.images.data(), flat.images.data(), &in.geometry,
                                     xs_spectrum_file_get(in.spectrum), &cc, (int32_t)in.materials.size(),
                                     in.materials.data(), vol.data(), stack.data(), reports.data(), 0));
    double voxel[3];
    xs_default_voxel_size(&in.geometry, dims, voxel); // REF correction.cpp:160
    check(xs_volume_file_save((c.output_dir / "corrected.xvol").string().c_str(), dims, voxel, vol.data()),
          lib_error);
    check(xs_stack_file_save((c.output_dir / "corrected.xprj").string().c_str(), raw.nu, raw.nv, raw.n,
                             stack.data()),
          lib_error);
    { // REF write_reports (correction.cpp:88-108)
        std::ofstream out(c.output_dir / "iterations.txt");
        if (!out)
            throw Failure{"cannot write report " + (c.output_dir / "iterations.txt").string()};
        for (int k = 0; k < n_it; ++k) {
            const xs_iteration_report& r = reports[k];
            out << "iteration=" << r.iteration << "\n"
                << "seconds_fbp=" << r.seconds_fbp << "\n"
                << "seconds_segmentation=" << r.seconds_segmentation << "\n"
                << "seconds_mc_scatter=" << r.seconds_mc_scatter << "\n"
                << "seconds_mc_primary=" << r.seconds_mc_primary << "\n"
                << "seconds_postprocess=" << r.seconds_postprocess << "\n"
                << "seconds_correction=" << r.seconds_correction << "\n"
                << "seconds_total=" << r.seconds_total << "\n"
                << "mc_seconds_per_projection=" << r.mc_seconds_per_projection << "\n"
                << "mean_scatter_fraction=" << r.mean_scatter_fraction << "\n"
                << "ncc_to_previous=" << r.ncc_to_previous << "\n"
                << "negative_scatter_clamped=" << r.negative_scatter_clamped << "\n\n";
        }
    }
    { // REF write_summary_csv (correction.cpp:110-123)
        std::ofstream out(c.output_dir / "summary.csv");
        if (!out)
            throw Failure{"cannot write summary " + (c.output_dir / "summary.csv").string()};
        out << "iteration,photons,splitting,step_size,mc_time_per_projection_s,"
               "mc_time_per_iteration_s,correction_time_per_iteration_s\n";
        for (int k = 0; k < n_it; ++k) {
            const xs_iteration_report& r = reports[k];
            out << r.iteration << "," << c.sim.photons_total << "," << c.sim.splitting << "," << c.sim.step_voxels
                << "," << r.mc_seconds_per_projection << "," << (r.seconds_mc_scatter + r.seconds_mc_primary) << ","
                << r.seconds_total << "\n";
        }
    }
    for (int k = 0; k < n_it; ++k)
        std::printf("iteration %d: %.1f s total, %.3f s/projection MC, scatter fraction %.3f, NCC %.5f\n",
                    reports[k].iteration, reports[k].seconds_total, reports[k].mc_seconds_per_projection,
                    reports[k].mean_scatter_fraction, reports[k].ncc_to_previous);
    return 0;
}

// ------------------------------------------------------ synthetic phantoms
// REF synthetic.cpp:20-117 (the same generators as paper_2201_13191_b200/
// synthetic.py): voxel centres origin + (i + 1/2) h, a voxel is inside a
// cylinder when dx^2 + dy^2 <= r^2 and |z| <= half height.
struct Phantom {
    int n = 0;
    double vs = 0.0, origin = 0.0;
    std::vector<uint8_t> ids;
    std::vector<float> dens;
    double centre(int i) const { return origin + (i + 0.5) * vs; }
};

Phantom empty_phantom(int n, double vs)
{
    if (n <= 0) // REF validate_phantom
        throw Failure{"phantom: dims must be positive"};
    if (!(vs > 0.0))
        throw Failure{"phantom: voxel size must be positive"};
    Phantom p;
    p.n = n;
    p.vs = vs;
    p.origin = (-n * vs) * 0.5;
    p.ids.assign((size_t)n * n * n, 0);
    p.dens.assign((size_t)n * n * n, 0.0f);
    return p;
}

void fill_cylinder(Phantom& p, double cx, double cy, double r, double half, uint8_t id, double density)
{
    const double r2 = r * r;
    for (int iz = 0; iz < p.n; ++iz) {
        if (!(std::abs(p.centre(iz)) <= half))
            continue;
        for (int iy = 0; iy < p.n; ++iy) {
            const double dy = p.centre(iy) - cy;
            for (int ix = 0; ix < p.n; ++ix) {
                const double dx = p.centre(ix) - cx;
                if (dx * dx + dy * dy <= r2) {
                    const size_t v = (size_t)ix + (size_t)p.n * ((size_t)iy + (size_t)p.n * iz);
                    p.ids[v] = id;
                    p.dens[v] = (float)density;
                }
            }
        }
    }
}

int cmd_phantom(const std::string& kind, const std::string& out, int dim, double vcm, const std::string& mdir,
                double radius, double height, int n_rods)
{
    const double kPi = 3.14159265358979323846;
    std::vector<xs_material_file*> files;
    struct Free {
        std::vector<xs_material_file*>& f;
        ~Free()
        {
            for (auto* x : f)
                xs_material_file_free(x);
        }
    } free_files{files};
    auto mat = [&](const char* name) -> const xs_material& {
        xs_material_file* f = nullptr;
        check(xs_material_file_load((fs::path(mdir) / name).string().c_str(), &f), lib_error);
        files.push_back(f);
        return *xs_material_file_get(f);
    };
    Phantom p;
    std::vector<xs_material> mats(1);
    mats[0].name = "vacuum";
    if (kind == "empty") { // simulate --what primary on it gives the flat field
        mats.push_back(mat("water.mat"));
        p = empty_phantom(dim, vcm);
    } else if (kind == "cube") {
        mats.push_back(mat("water.mat"));
        const double edge = radius > 0 ? 2.0 * radius : dim * vcm * 0.5;
        if (!(edge > 0.0))
            throw Failure{"cube phantom: edge must be > 0"};
        p = empty_phantom(dim, vcm);
        const double half = 0.5 * edge;
        for (int iz = 0; iz < dim; ++iz)
            for (int iy = 0; iy < dim; ++iy)
                for (int ix = 0; ix < dim; ++ix)
                    if (std::abs(p.centre(iz)) <= half && std::abs(p.centre(iy)) <= half &&
                        std::abs(p.centre(ix)) <= half) {
                        const size_t v = (size_t)ix + (size_t)dim * ((size_t)iy + (size_t)dim * iz);
                        p.ids[v] = 1;
                        p.dens[v] = 1.0f;
                    }
    } else if (kind == "cylinder") {
        mats.push_back(mat("water.mat"));
        if (!(radius > 0.0 && height > 0.0))
            throw Failure{"cylinder phantom: radius and height must be > 0"};
        p = empty_phantom(dim, vcm);
        fill_cylinder(p, 0.0, 0.0, radius, 0.5 * height, 1, 1.0);
    } else if (kind == "rods") {
        const xs_material& body = mat("cement.mat");
        const xs_material& rod = mat("iron.mat");
        mats.push_back(body);
        mats.push_back(rod);
        const double rod_r = radius * 0.08, ring_r = radius * 0.6;
        if (!(radius > 0.0 && rod_r > 0.0))
            throw Failure{"rods phantom: radii must be > 0"};
        if (n_rods < 1)
            throw Failure{"rods phantom: need at least one rod"};
        if (ring_r + rod_r > radius)
            throw Failure{"rods phantom: rods extend outside the body"};
        p = empty_phantom(dim, vcm);
        fill_cylinder(p, 0.0, 0.0, radius, 0.5 * height, 1, body.density_ref);
        for (int k = 0; k < n_rods; ++k) {
            const double phi = 2.0 * kPi * k / n_rods;
            fill_cylinder(p, ring_r * std::cos(phi), ring_r * std::sin(phi), rod_r, 0.5 * height, 2, rod.density_ref);
        }
    } else if (kind == "cylinder-head-like") {
        const xs_material& body = mat("aluminum.mat");
        const xs_material& insert = mat("iron.mat");
        mats.push_back(body);
        mats.push_back(insert);
        p = empty_phantom(dim, vcm);
        const double extent = dim * vcm, body_r = 0.42 * extent, half = 0.5 * (0.8 * extent);
        fill_cylinder(p, 0.0, 0.0, body_r, half, 1, body.density_ref);
        for (int k = 0; k < 4; ++k) { // four air bores
            const double phi = 2.0 * kPi * (k + 0.5) / 4.0;
            fill_cylinder(p, 0.55 * body_r * std::cos(phi), 0.55 * body_r * std::sin(phi), 0.18 * body_r, half * 0.9, 0,
                          0.0);
        }
        for (int k = 0; k < 8; ++k) { // a ring of eight dense inserts
            const double phi = 2.0 * kPi * k / 8.0;
            fill_cylinder(p, 0.8 * body_r * std::cos(phi), 0.8 * body_r * std::sin(phi), 0.07 * body_r, half * 0.8, 2,
                          insert.density_ref);
        }
    } else {
        std::cerr << "unknown phantom kind '" << kind << "' (empty|cube|cylinder|rods|cylinder-head-like)\n";
        return kExitValidation;
    }
    xs_phantom ph{};
    ph.dims[0] = ph.dims[1] = ph.dims[2] = dim;
    ph.voxel_size[0] = ph.voxel_size[1] = ph.voxel_size[2] = vcm;
    ph.origin[0] = ph.origin[1] = ph.origin[2] = p.origin;
    ph.material_id = p.ids.data();
    ph.density = p.dens.data();
    ph.n_materials = (int32_t)mats.size();
    ph.materials = mats.data();
    check(xs_validate_phantom(&ph), lib_error);
    check(xs_phantom_file_save(out.c_str(), &ph), lib_error);
    std::printf("wrote %s (%d^3 voxels of %.3f cm)\n", out.c_str(), dim, vcm);
    return 0;
}

// ----------------------------------------------------------------- metrics
// REF metrics.cpp (mse, ncc with population statistics, cnr, profile_line)
// over one image of a stack (.xprj) or a volume slice (.xvol).
struct Image {
    int nu = 0, nv = 0;
    std::vector<double> v;
    double at(int c, int r) const { return v[(size_t)r * nu + c]; }
};

Image load_image(const std::string& path, int slice)
{
    Image img;
    if (path.size() >= 5 && path.compare(path.size() - 5, 5, ".xvol") == 0) {
        int32_t d[3];
        double vs[3];
        check(xs_volume_file_info(path.c_str(), d, vs), lib_error);
        std::vector<float> vol((size_t)d[0] * d[1] * d[2]);
        check(xs_volume_file_load(path.c_str(), vol.data()), lib_error);
        const int iz = slice < 0 ? d[2] / 2 : slice;
        if (iz < 0 || iz >= d[2])
            throw Failure{"volume_slice_z: slice index out of range"};
        img.nu = d[0];
        img.nv = d[1];
        img.v.assign(vol.begin() + (size_t)iz * d[0] * d[1], vol.begin() + (size_t)(iz + 1) * d[0] * d[1]);
        return img;
    }
    const Stack st = load_stack(path, {});
    const int k = slice < 0 ? 0 : slice;
    if (k >= st.n)
        throw Failure{"vector::_M_range_check: __n (which is " + std::to_string(k) + ") >= this->size() (which is " +
                      std::to_string(st.n) + ")"};
    img.nu = st.nu;
    img.nv = st.nv;
    const size_t np = (size_t)st.nu * st.nv;
    img.v.assign(st.images.begin() + (size_t)k * np, st.images.begin() + (size_t)(k + 1) * np);
    return img;
}

double mean_of(const std::vector<double>& x)
{
    double s = 0.0;
    for (double v : x)
        s += v;
    return s / x.size();
}

int cmd_metrics(const std::string& a_path, const std::string& b_path, const std::string& roi, int slice,
                const std::string& out_csv, const std::string& profile, const std::string& profile_out)
{
    const Image a = load_image(a_path, slice);
    std::ostringstream csv;
    csv << "metric,value\n";
    if (!b_path.empty()) {
        const Image b = load_image(b_path, slice);
        if (a.nu != b.nu || a.nv != b.nv)
            throw Failure{"mse: image dims mismatch"};
        if (a.v.empty())
            throw Failure{"mse: size mismatch"};
        double s = 0.0;
        for (size_t i = 0; i < a.v.size(); ++i) {
            const double d = a.v[i] - b.v[i];
            s += d * d;
        }
        csv << "mse," << s / a.v.size() << "\n";
        const double m1 = mean_of(a.v), m2 = mean_of(b.v);
        double cov = 0.0, v1 = 0.0, v2 = 0.0;
        for (size_t i = 0; i < a.v.size(); ++i) {
            const double x = a.v[i] - m1, y = b.v[i] - m2;
            cov += x * y;
            v1 += x * x;
            v2 += y * y;
        }
        if (!(v1 > 0.0) || !(v2 > 0.0))
            throw Failure{"ncc: zero variance input"};
        csv << "ncc," << cov / std::sqrt(v1 * v2) << "\n";
    }
    if (!roi.empty()) {
        int q[8];
        if (std::sscanf(roi.c_str(), "%d,%d,%d,%d,%d,%d,%d,%d", &q[0], &q[1], &q[2], &q[3], &q[4], &q[5], &q[6],
                        &q[7]) != 8) {
            std::cerr << "--roi wants roi_row,roi_col,h,w,bg_row,bg_col,h,w\n";
            return kExitValidation;
        }
        auto rect = [&](int row, int col, int h, int w, const char* what) {
            if (row < 0 || col < 0 || h <= 0 || w <= 0 || row + h > a.nv || col + w > a.nu)
                throw Failure{std::string("cnr: ") + what + " rectangle outside image"};
        };
        rect(q[0], q[1], q[2], q[3], "ROI");
        rect(q[4], q[5], q[6], q[7], "background");
        if (q[0] < q[4] + q[6] && q[4] < q[0] + q[2] && q[1] < q[5] + q[7] && q[5] < q[1] + q[3])
            throw Failure{"cnr: ROI and background rectangles overlap"};
        double rs = 0.0;
        for (int r = q[0]; r < q[0] + q[2]; ++r)
            for (int c = q[1]; c < q[1] + q[3]; ++c)
                rs += a.at(c, r);
        const double roi_mean = rs / (static_cast<double>(q[2]) * q[3]);
        double bs = 0.0;
        const double bn = static_cast<double>(q[6]) * q[7];
        for (int r = q[4]; r < q[4] + q[6]; ++r)
            for (int c = q[5]; c < q[5] + q[7]; ++c)
                bs += a.at(c, r);
        const double bg_mean = bs / bn;
        double bv = 0.0;
        for (int r = q[4]; r < q[4] + q[6]; ++r)
            for (int c = q[5]; c < q[5] + q[7]; ++c) {
                const double d = a.at(c, r) - bg_mean;
                bv += d * d;
            }
        bv /= bn;
        if (!(bv > 0.0))
            throw Failure{"cnr: zero background standard deviation"};
        csv << "cnr," << std::abs(roi_mean - bg_mean) / std::sqrt(bv) << "\n";
    }
    if (!profile.empty()) { // a row band averaged per column
        int r0 = 0, r1 = 0, c0 = 0, c1 = a.nu;
        const int k = std::sscanf(profile.c_str(), "%d,%d,%d,%d", &r0, &r1, &c0, &c1);
        if (k != 2 && k != 4) {
            std::cerr << "--profile wants row0,row1[,col0,col1]\n";
            return kExitValidation;
        }
        if (k == 2) {
            c0 = 0;
            c1 = a.nu;
        }
        if (r0 < 0 || c0 < 0 || r1 > a.nv || c1 > a.nu || r0 >= r1 || c0 >= c1)
            throw Failure{"profile_line: empty or out-of-bounds range"};
        std::ofstream pout(profile_out.empty() ? "profile.csv" : profile_out);
        pout << "column,value\n";
        for (int c = c0; c < c1; ++c) {
            double sum = 0.0;
            for (int r = r0; r < r1; ++r)
                sum += a.at(c, r);
            pout << c << "," << sum / (r1 - r0) << "\n";
        }
    }
    if (out_csv.empty()) {
        std::cout << csv.str();
    } else {
        std::ofstream o(out_csv);
        o << csv.str();
    }
    return 0;
}

bool ends_with(const std::string& s, const char* suf)
{
    const size_t k = std::char_traits<char>::length(suf);
    return s.size() >= k && s.compare(s.size() - k, k, suf) == 0;
}

int cmd_inspect(const std::string& path, int slice, const std::string& out)
{
    if (ends_with(path, ".xvox")) {
        int32_t d[3];
        double vs[3], o[3];
        uint32_t nm = 0;
        check(xs_phantom_file_info(path.c_str(), d, vs, o, &nm), lib_error);
        std::printf("XVOX1 phantom: dims %d x %d x %d, voxel %.4f x %.4f x %.4f cm, "
                    "origin (%.3f, %.3f, %.3f), %u materials\n",
                    d[0], d[1], d[2], vs[0], vs[1], vs[2], o[0], o[1], o[2], nm);
    } else if (ends_with(path, ".xprj")) {
        int32_t nu = 0, nv = 0, na = 0;
        check(xs_stack_file_info(path.c_str(), &nu, &nv, &na), lib_error);
        std::vector<double> img((size_t)nu * nv * na);
        check(xs_stack_file_load(path.c_str(), img.data()), lib_error); // (REF loads the stack)
        std::printf("XPRJ1 stack: %d x %d pixels, %d angles\n", nu, nv, na);
    } else if (ends_with(path, ".xvol")) {
        int32_t d[3];
        double vs[3];
        check(xs_volume_file_info(path.c_str(), d, vs), lib_error);
        std::vector<float> v((size_t)d[0] * d[1] * d[2]);
        check(xs_volume_file_load(path.c_str(), v.data()), lib_error);
        std::printf("XVOL1 volume: dims %d x %d x %d, voxel %.4f x %.4f x %.4f cm\n", d[0], d[1], d[2], vs[0],
                    vs[1], vs[2]);
        if (!out.empty()) {
            const int iz = slice < 0 ? d[2] / 2 : slice;
            if (iz < 0 || iz >= d[2]) // REF volume_slice_z
                throw Failure{"volume_slice_z: slice index out of range"};
            const size_t plane = (size_t)d[0] * d[1];
            const float* s = v.data() + (size_t)iz * plane;
            if (ends_with(out, ".csv")) { // REF save_slice_csv
                std::ofstream f(out);
                if (!f)
                    throw Failure{"cannot write " + out};
                for (int y = 0; y < d[1]; ++y)
                    for (int x = 0; x < d[0]; ++x)
                        f << (double)s[(size_t)y * d[0] + x] << (x + 1 == d[0] ? '\n' : ',');
            } else { // REF save_slice_pgm, range from the slice
                double lo = *std::min_element(s, s + plane), hi = *std::max_element(s, s + plane);
                if (!(hi > lo))
                    hi = lo + 1.0;
                std::ofstream f(out, std::ios::binary);
                if (!f)
                    throw Failure{"cannot write " + out};
                f << "P5\n" << d[0] << " " << d[1] << "\n255\n";
                for (size_t i = 0; i < plane; ++i) {
                    const double t = std::clamp(((double)s[i] - lo) / (hi - lo), 0.0, 1.0);
                    const unsigned char b = static_cast<unsigned char>(t * 255.0 + 0.5);
                    f.write(reinterpret_cast<const char*>(&b), 1);
                }
            }
            std::printf("wrote slice %d to %s\n", iz, out.c_str());
        }
    } else {
        std::cerr << "unknown file type (expected .xvox/.xprj/.xvol)\n";
        return kExitValidation;
    }
    return 0;
}

int usage(const std::string& why)
{
    std::cerr << why << "\n"
              << "usage: xscat_b200 simulate --config FILE [--what primary|scatter|both] [--angles a:b|i,j,...]\n"
              << "                            [--seed N] [--threads N]\n"
              << "       xscat_b200 reconstruct --config FILE --stack S.xprj [--flat F.xprj] --out V.xvol [--dim N]\n"
              << "       xscat_b200 correct --config FILE --raw R.xprj --flat F.xprj [--seed N] [--threads N]\n"
              << "       xscat_b200 phantom --kind KIND --out P.xvox [--dim N] [--voxel-cm X] [--radius-cm R]\n"
              << "                          [--height-cm H] [--rods K] [--materials-dir D]\n"
              << "       xscat_b200 metrics --a A [--b B] [--roi r,c,h,w,br,bc,bh,bw] [--slice N] [--out CSV]\n"
              << "                          [--profile r0,r1[,c0,c1]] [--profile-out CSV]\n"
              << "       xscat_b200 inspect --file FILE [--slice N] [--export out.pgm|out.csv]\n";
    return kExitValidation;
}

} // namespace

int main(int argc, char** argv)
{
    if (argc < 2)
        return usage("a subcommand is required");
    const std::string cmd = argv[1];
    std::map<std::string, std::string> opt;
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0)
            return usage("unexpected argument: " + a);
        std::string value;
        if (const size_t eq = a.find('='); eq != std::string::npos) {
            value = a.substr(eq + 1);
            a = a.substr(0, eq);
        } else if (i + 1 < argc) {
            value = argv[++i];
        } else {
            return usage(a + ": missing value");
        }
        opt[a] = value;
    }
    auto allowed = [&](std::initializer_list<const char*> names) -> std::string {
        for (const auto& [k, v] : opt)
            if (std::none_of(names.begin(), names.end(), [&](const char* n) { return k == n; }))
                return k;
        return "";
    };
    try {
        Flags flags;
        try {
            if (opt.count("--seed"))
                flags.seed = std::stoull(opt["--seed"]);
            if (opt.count("--threads"))
                flags.threads = std::stoi(opt["--threads"]);
        } catch (const std::exception&) {
            return usage("--seed / --threads: not a number");
        }
        if (cmd == "simulate") {
            if (const std::string bad = allowed({"--config", "--seed", "--threads", "--what", "--angles"}); !bad.empty())
                return usage("simulate: unknown option " + bad);
            if (!opt.count("--config"))
                return usage("simulate: --config is required");
            flags.config = opt["--config"];
            return cmd_simulate(flags, opt.count("--what") ? opt["--what"] : "both", opt["--angles"],
                                opt.count("--angles") > 0);
        }
        if (cmd == "reconstruct") {
            if (const std::string bad = allowed({"--config", "--seed", "--threads", "--stack", "--flat", "--out", "--dim"});
                !bad.empty())
                return usage("reconstruct: unknown option " + bad);
            if (!opt.count("--config") || !opt.count("--stack") || !opt.count("--out"))
                return usage("reconstruct: --config, --stack and --out are required");
            flags.config = opt["--config"];
            return cmd_reconstruct(flags, opt["--stack"], opt["--flat"], opt["--out"],
                                   opt.count("--dim") ? std::stoi(opt["--dim"]) : 64);
        }
        if (cmd == "correct") {
            if (const std::string bad = allowed({"--config", "--seed", "--threads", "--raw", "--flat"}); !bad.empty())
                return usage("correct: unknown option " + bad);
            if (!opt.count("--config") || !opt.count("--raw") || !opt.count("--flat"))
                return usage("correct: --config, --raw and --flat are required");
            flags.config = opt["--config"];
            return cmd_correct(flags, opt["--raw"], opt["--flat"]);
        }
        if (cmd == "phantom") {
            if (const std::string bad = allowed({"--kind", "--out", "--dim", "--voxel-cm", "--radius-cm", "--height-cm",
                                                 "--rods", "--materials-dir", "--seed", "--threads"});
                !bad.empty())
                return usage("phantom: unknown option " + bad);
            if (!opt.count("--kind") || !opt.count("--out"))
                return usage("phantom: --kind and --out are required");
            auto num = [&](const char* k, double d) { return opt.count(k) ? std::stod(opt[k]) : d; };
            return cmd_phantom(opt["--kind"], opt["--out"], opt.count("--dim") ? std::stoi(opt["--dim"]) : 64,
                               num("--voxel-cm", 0.2),
                               opt.count("--materials-dir") ? opt["--materials-dir"] : "data/materials",
                               num("--radius-cm", 4.0), num("--height-cm", 10.0),
                               opt.count("--rods") ? std::stoi(opt["--rods"]) : 8);
        }
        if (cmd == "metrics") {
            if (const std::string bad = allowed({"--a", "--b", "--roi", "--slice", "--out", "--profile", "--profile-out",
                                                 "--seed", "--threads"});
                !bad.empty())
                return usage("metrics: unknown option " + bad);
            if (!opt.count("--a"))
                return usage("metrics: --a is required");
            return cmd_metrics(opt["--a"], opt["--b"], opt["--roi"], opt.count("--slice") ? std::stoi(opt["--slice"]) : -1,
                               opt["--out"], opt["--profile"], opt["--profile-out"]);
        }
        if (cmd == "inspect") {
            if (const std::string bad = allowed({"--file", "--slice", "--export", "--seed", "--threads"}); !bad.empty())
                return usage("inspect: unknown option " + bad);
            if (!opt.count("--file"))
                return usage("inspect: --file is required");
            return cmd_inspect(opt["--file"], opt.count("--slice") ? std::stoi(opt["--slice"]) : -1, opt["--export"]);
        }
        return usage("unknown subcommand '" + cmd + "' (simulate, reconstruct, correct, phantom, metrics, inspect)");
    } catch (const Failure& e) {
        std::cerr << "error: " << e.msg << "\n";
        return kExitRuntime;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitRuntime;
    }
}
