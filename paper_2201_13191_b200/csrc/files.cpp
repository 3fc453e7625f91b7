// files.cpp — the reference's file formats and input loaders, host side of
// libxscatgpu.so (no GPU needed).  SURVEY.md §8(f) rank 4.
//
//   XPRJ1 projection stacks   REF detector_image.cpp:33-87
//   XVOX1 voxel phantoms      REF phantom.cpp:74-161
//   XVOL1 volumes             REF volume.cpp:22-62
//   material tables (.mat)    REF material.cpp:57-97 (validation), :129-213
//   spectra (keV, weight)     REF spectrum.cpp:11-60
//   detector response         REF detector_response.cpp:11-20, :50-79
//
// Byte layouts, accepted inputs and error messages are the reference's, so a
// file either program writes loads in the other and a bad file fails with
// the same text (tests/test_files.py against files the compiled reference
// wrote).  Numbers are parsed with the same standard-library conversions the
// reference uses (std::stod for header values, stream extraction for table
// rows), so every table value is the identical double.
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_common.h"

using xsh::Error;

namespace {

template <typename F>
int run(F&& f)
{
    try {
        f();
        return XS_OK;
    } catch (const Error& e) {
        return xsh::set_error(e.code, e.msg);
    } catch (const std::exception& e) {
        return xsh::set_error(XS_E_RUNTIME, e.what());
    }
}

[[noreturn]] void raise(const std::string& msg) { throw Error{XS_E_RUNTIME, msg}; }

// the string without leading / trailing white space (the C locale's isspace set)
std::string trim(const std::string& s)
{
    static const char* const ws = " \t\n\v\f\r";
    const size_t first = s.find_first_not_of(ws);
    return first == std::string::npos ? std::string() : s.substr(first, s.find_last_not_of(ws) + 1 - first);
}

// text line without its '#' comment
std::string uncomment(std::string line)
{
    const size_t h = line.find('#');
    if (h != std::string::npos)
        line.erase(h);
    return line;
}

template <typename T>
void put(std::ofstream& out, const T& v)
{
    out.write(reinterpret_cast<const char*>(&v), sizeof v);
}

template <typename T>
void get(std::ifstream& in, T& v)
{
    in.read(reinterpret_cast<char*>(&v), sizeof v);
}

void expect_magic(std::ifstream& in, const std::string& path, const char* magic)
{
    char m[5];
    in.read(m, 5);
    if (!in || std::memcmp(m, magic, 5) != 0)
        raise(path + ": bad magic (expected " + magic + ")");
}

// ---------------------------------------------------------------- XPRJ1
// "XPRJ1", u32 nu, nv, n_angles, then n_angles images of nu*nv f32 (row-major)
struct StackHeader {
    uint32_t nu, nv, n;
};

StackHeader stack_header(std::ifstream& in, const std::string& path)
{
    if (!in)
        raise("cannot open projection stack " + path);
    expect_magic(in, path, "XPRJ1");
    StackHeader h{};
    uint32_t w[3];
    in.read(reinterpret_cast<char*>(w), sizeof w);
    if (!in)
        raise(path + ": truncated header");
    h.nu = w[0];
    h.nv = w[1];
    h.n = w[2];
    return h;
}

// ---------------------------------------------------------------- XVOX1
// "XVOX1", u32 nx, ny, nz, f64 voxel[3], f64 origin[3], u32 n_materials,
// nx*ny*nz u8 ids, nx*ny*nz f32 densities
struct PhantomHeader {
    uint32_t d[3];
    double voxel[3], origin[3];
    uint32_t n_materials;
};

PhantomHeader phantom_header(std::ifstream& in, const std::string& path)
{
    if (!in)
        raise("cannot open phantom file " + path);
    expect_magic(in, path, "XVOX1");
    PhantomHeader h{};
    for (auto& v : h.d)
        get(in, v);
    for (auto& v : h.voxel)
        get(in, v);
    for (auto& v : h.origin)
        get(in, v);
    get(in, h.n_materials);
    if (!in)
        raise(path + ": truncated header");
    return h;
}

// ---------------------------------------------------------------- XVOL1
// "XVOL1", u32 nx, ny, nz, f64 voxel[3], nx*ny*nz f32 values (x fastest)
struct VolumeHeader {
    uint32_t d[3];
    double voxel[3];
};

VolumeHeader volume_header(std::ifstream& in, const std::string& path)
{
    if (!in)
        raise("cannot open volume " + path);
    expect_magic(in, path, "XVOL1");
    VolumeHeader h{};
    in.read(reinterpret_cast<char*>(h.d), sizeof h.d);
    for (auto& v : h.voxel)
        get(in, v);
    // (the reference reads the voxel size without a header check; a short
    // file fails at the data read below)
    return h;
}

uint64_t count3(const uint32_t* d) { return (uint64_t)d[0] * d[1] * d[2]; }

} // namespace

struct xs_phantom_file {
    std::vector<uint8_t> ids;
    std::vector<float> dens;
    xs_phantom view;
};

// ------------------------------------------------------------ text tables
struct xs_material_file {
    std::string name;
    std::vector<double> x[6], y[6];
    xs_material view;
};

struct xs_spectrum_file {
    std::vector<double> e, w;
    xs_spectrum view;
};

struct xs_response_file {
    std::vector<double> e, dqe, dep;
    xs_response view;
};

namespace {

const char* const kSections[6] = {"mu", "incoherent", "coherent", "photoelectric", "S", "F"};

[[noreturn]] void parse_error(const std::string& path, int line, const std::string& what)
{
    raise(path + ":" + std::to_string(line) + ": parse error: " + what);
}

[[noreturn]] void invariant(const std::string& name, const std::string& what)
{
    raise("material '" + name + "': invariant violation: " + what);
}

// REF load_material's table pick-up (material.cpp:195-209: present, increasing
// abscissa, in section order), then validate_material (:57-97), in its order
void check_material(const xs_material_file& f, double z_eff, double density)
{
    const std::string& n = f.name;
    for (int t = 0; t < 6; ++t) {
        if (f.x[t].empty())
            invariant(n, std::string("missing table [") + kSections[t] + "]");
        for (size_t i = 1; i < f.x[t].size(); ++i)
            if (!(f.x[t][i] > f.x[t][i - 1]))
                invariant(n, std::string("non-monotone abscissa in [") + kSections[t] + "]");
    }
    if (n.empty())
        invariant("(unnamed)", "missing name");
    if (!(z_eff > 0.0))
        invariant(n, "z_eff must be > 0");
    if (!(density > 0.0))
        invariant(n, "density must be > 0");
    for (int t = 0; t < 6; ++t) {
        const auto& x = f.x[t];
        const auto& y = f.y[t];
        if (x.empty())
            invariant(n, std::string("missing table [") + kSections[t] + "]");
        for (size_t i = 1; i < x.size(); ++i)
            if (!(x[i] > x[i - 1]))
                invariant(n, std::string("non-monotone abscissa in [") + kSections[t] + "]");
        for (double v : y)
            if (!(v >= 0.0) || !std::isfinite(v))
                invariant(n, std::string("negative or non-finite value in [") + kSections[t] + "]");
    }
    for (double v : f.y[0])
        if (!(v > 0.0))
            invariant(n, "mu values must be > 0");
    const auto &sq = f.x[4], &sv = f.y[4];
    if (sq.front() != 0.0 || sv.front() != 0.0)
        invariant(n, "S table must start at S(0) = 0");
    for (size_t i = 1; i < sv.size(); ++i)
        if (sv[i] < sv[i - 1])
            invariant(n, "S must be non-decreasing in q");
    if (sv.back() > z_eff * (1.0 + 1e-9))
        invariant(n, "S must not exceed z_eff");
    const auto &fq = f.x[5], &fv = f.y[5];
    if (fq.front() != 0.0)
        invariant(n, "F table must start at q = 0");
    if (std::abs(fv.front() - z_eff) > 1e-9 * z_eff)
        invariant(n, "F(0) must equal z_eff");
    for (size_t i = 1; i < fv.size(); ++i)
        if (fv[i] > fv[i - 1] * (1.0 + 1e-12) + 1e-15)
            invariant(n, "F must be non-increasing in q");
}

// two- or three-column numeric CSV ('#' comments, commas or blanks)
template <int N>
void read_columns(const std::string& path, const char* what_open, const char* what_cols,
                  std::vector<double> (&cols)[N])
{
    std::ifstream in(path);
    if (!in)
        raise(std::string("cannot open ") + what_open + " file " + path);
    std::string line;
    int no = 0;
    while (std::getline(in, line)) {
        ++no;
        line = uncomment(line);
        for (char& c : line)
            if (c == ',')
                c = ' ';
        std::istringstream row(line);
        double v[N] = {};
        if (!(row >> v[0]))
            continue; // blank line
        bool ok = true;
        for (int k = 1; k < N && ok; ++k)
            ok = static_cast<bool>(row >> v[k]);
        if (!ok)
            raise(path + ":" + std::to_string(no) + ": expected " + what_cols);
        for (int k = 0; k < N; ++k)
            cols[k].push_back(v[k]);
    }
}

} // namespace

extern "C" {

// ------------------------------------------------------------------ XPRJ1
int xs_stack_file_info(const char* path, int32_t* nu, int32_t* nv, int32_t* n_angles)
{
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        const StackHeader h = stack_header(in, path);
        *nu = (int32_t)h.nu;
        *nv = (int32_t)h.nv;
        *n_angles = (int32_t)h.n;
    });
}

int xs_stack_file_load(const char* path, double* images)
{
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        const StackHeader h = stack_header(in, path);
        const size_t np = (size_t)h.nu * h.nv;
        std::vector<float> buf(np);
        for (uint32_t a = 0; a < h.n; ++a) {
            in.read(reinterpret_cast<char*>(buf.data()), np * sizeof(float));
            if (!in)
                raise(std::string(path) + ": truncated pixel data");
            double* img = images + (size_t)a * np;
            for (size_t i = 0; i < np; ++i)
                img[i] = buf[i];
        }
    });
}

int xs_stack_file_save(const char* path, int32_t nu, int32_t nv, int32_t n_angles, const double* images)
{
    return run([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out)
            raise(std::string("cannot write projection stack ") + path);
        out.write("XPRJ1", 5);
        const uint32_t w[3] = {(uint32_t)nu, (uint32_t)nv, (uint32_t)n_angles};
        out.write(reinterpret_cast<const char*>(w), sizeof w);
        const size_t np = (size_t)nu * nv;
        std::vector<float> buf(np);
        for (int32_t a = 0; a < n_angles; ++a) {
            const double* img = images + (size_t)a * np;
            for (size_t i = 0; i < np; ++i)
                buf[i] = (float)img[i];
            out.write(reinterpret_cast<const char*>(buf.data()), np * sizeof(float));
        }
        if (!out)
            raise(std::string("write failed for ") + path);
    });
}

// ------------------------------------------------------------------ XVOX1
int xs_phantom_file_info(const char* path, int32_t dims[3], double voxel_size[3], double origin[3],
                         uint32_t* n_materials)
{
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        const PhantomHeader h = phantom_header(in, path);
        for (int a = 0; a < 3; ++a) {
            dims[a] = (int32_t)h.d[a];
            voxel_size[a] = h.voxel[a];
            origin[a] = h.origin[a];
        }
        *n_materials = h.n_materials;
    });
}

// REF load_phantom reads the header without a check of its own: a short
// header surfaces as truncated voxel data
int xs_phantom_file_read(const char* path, uint32_t n_materials_given, xs_phantom_file** out)
{
    *out = nullptr;
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in)
            raise(std::string("cannot open phantom file ") + path);
        expect_magic(in, path, "XVOX1");
        PhantomHeader h{};
        for (auto& v : h.d)
            get(in, v);
        for (auto& v : h.voxel)
            get(in, v);
        for (auto& v : h.origin)
            get(in, v);
        get(in, h.n_materials);
        // the caller's list (vacuum first) must cover the header's count
        if (n_materials_given < h.n_materials)
            raise(std::string(path) + ": header declares " + std::to_string(h.n_materials) +
                  " materials, only " + std::to_string(n_materials_given) + " provided");
        // (more voxels than the file holds -- or a product past 64 bits -- : the
        // read below would fail)
        if ((double)h.d[0] * (double)h.d[1] * (double)h.d[2] > 1e15)
            raise(std::string(path) + ": truncated voxel data");
        const uint64_t n = count3(h.d);
        std::streamoff left = 0;
        if (in) {
            const std::streamoff at = in.tellg();
            in.seekg(0, std::ios::end);
            left = in.tellg() - at;
            in.seekg(at);
        }
        if (!in || (uint64_t)left < n * 5)
            raise(std::string(path) + ": truncated voxel data");
        auto f = std::make_unique<xs_phantom_file>();
        f->ids.resize(n);
        f->dens.resize(n);
        in.read(reinterpret_cast<char*>(f->ids.data()), (std::streamsize)n);
        in.read(reinterpret_cast<char*>(f->dens.data()), (std::streamsize)(n * sizeof(float)));
        if (!in)
            raise(std::string(path) + ": truncated voxel data");
        xs_phantom& p = f->view;
        for (int a = 0; a < 3; ++a) {
            p.dims[a] = (int32_t)h.d[a];
            p.voxel_size[a] = h.voxel[a];
            p.origin[a] = h.origin[a];
        }
        p.material_id = f->ids.data();
        p.density = f->dens.data();
        p.n_materials = 0;
        p.materials = nullptr;
        *out = f.release();
    });
}

const xs_phantom* xs_phantom_file_get(const xs_phantom_file* f) { return f ? &f->view : nullptr; }
void xs_phantom_file_free(xs_phantom_file* f) { delete f; }

int xs_phantom_file_save(const char* path, const xs_phantom* ph)
{
    return run([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out)
            raise(std::string("cannot write phantom file ") + path);
        out.write("XVOX1", 5);
        for (int a = 0; a < 3; ++a)
            put(out, (uint32_t)ph->dims[a]);
        for (int a = 0; a < 3; ++a)
            put(out, ph->voxel_size[a]);
        for (int a = 0; a < 3; ++a)
            put(out, ph->origin[a]);
        put(out, (uint32_t)ph->n_materials);
        const uint64_t n = (uint64_t)ph->dims[0] * ph->dims[1] * ph->dims[2];
        out.write(reinterpret_cast<const char*>(ph->material_id), (std::streamsize)n);
        out.write(reinterpret_cast<const char*>(ph->density), (std::streamsize)(n * sizeof(float)));
        if (!out)
            raise(std::string("write failed for ") + path);
    });
}

// ------------------------------------------------------------------ XVOL1
int xs_volume_file_info(const char* path, int32_t dims[3], double voxel_size[3])
{
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        const VolumeHeader h = volume_header(in, path);
        for (int a = 0; a < 3; ++a) {
            dims[a] = (int32_t)h.d[a];
            voxel_size[a] = h.voxel[a];
        }
    });
}

int xs_volume_file_load(const char* path, float* values)
{
    return run([&] {
        std::ifstream in(path, std::ios::binary);
        const VolumeHeader h = volume_header(in, path);
        in.read(reinterpret_cast<char*>(values), (std::streamsize)(count3(h.d) * sizeof(float)));
        if (!in)
            raise(std::string(path) + ": truncated volume data");
    });
}

int xs_volume_file_save(const char* path, const int32_t dims[3], const double voxel_size[3], const float* values)
{
    return run([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out)
            raise(std::string("cannot write volume ") + path);
        out.write("XVOL1", 5);
        for (int a = 0; a < 3; ++a)
            put(out, (uint32_t)dims[a]);
        for (int a = 0; a < 3; ++a)
            put(out, voxel_size[a]);
        const uint64_t n = (uint64_t)dims[0] * dims[1] * dims[2];
        out.write(reinterpret_cast<const char*>(values), (std::streamsize)(n * sizeof(float)));
        if (!out)
            raise(std::string("write failed for ") + path);
    });
}

// REF validate_phantom (phantom.cpp:33-56) on the host, in its order
int xs_validate_phantom(const xs_phantom* ph)
{
    return run([&] {
        if (ph->dims[0] <= 0 || ph->dims[1] <= 0 || ph->dims[2] <= 0)
            raise("phantom: dims must be positive");
        if (!(ph->voxel_size[0] > 0.0 && ph->voxel_size[1] > 0.0 && ph->voxel_size[2] > 0.0))
            raise("phantom: voxel size must be positive");
        if (ph->n_materials <= 0 || !ph->materials)
            raise("phantom: no material table");
        const uint64_t n = (uint64_t)ph->dims[0] * ph->dims[1] * ph->dims[2];
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t id = ph->material_id[i];
            if (id >= (uint32_t)ph->n_materials)
                raise("phantom: material id " + std::to_string(id) + " has no loaded material");
            const xs_material& m = ph->materials[id];
            if (id != 0 && m.mu.n <= 0)
                raise("phantom: material id " + std::to_string(id) + " (" + (m.name ? m.name : "") +
                      ") has no tables");
            if (!(ph->density[i] >= 0.0f))
                raise("phantom: negative density");
            if (id == 0 && ph->density[i] != 0.0f)
                raise("phantom: vacuum voxel with nonzero density");
        }
    });
}

// ------------------------------------------------------- material tables
int xs_material_file_load(const char* path_c, xs_material_file** out)
{
    *out = nullptr;
    return run([&] {
        const std::string path = path_c;
        std::ifstream in(path);
        if (!in)
            raise("cannot open material file " + path);
        auto f = std::make_unique<xs_material_file>();
        double z_eff = 0.0, density = 0.0;
        bool has_name = false, has_z = false, has_density = false;
        int section = -1; // -1: header
        std::string line;
        int no = 0;
        while (std::getline(in, line)) {
            ++no;
            line = trim(uncomment(line));
            if (line.empty())
                continue;
            if (line.front() == '[') {
                if (line.back() != ']')
                    parse_error(path, no, "malformed section header");
                const std::string tag = trim(line.substr(1, line.size() - 2));
                section = -2;
                for (int t = 0; t < 6; ++t)
                    if (tag == kSections[t])
                        section = t;
                if (section == -2)
                    parse_error(path, no, "unknown section [" + tag + "]");
                continue;
            }
            if (section < 0) { // header: key = value
                const size_t eq = line.find('=');
                if (eq == std::string::npos)
                    parse_error(path, no, "expected key=value before first section");
                const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
                try {
                    if (key == "name") {
                        f->name = value;
                        has_name = true;
                    } else if (key == "z_eff") {
                        z_eff = std::stod(value);
                        has_z = true;
                    } else if (key == "density") {
                        density = std::stod(value);
                        has_density = true;
                    } else {
                        parse_error(path, no, "unknown header key '" + key + "'");
                    }
                } catch (const std::invalid_argument&) {
                    parse_error(path, no, "cannot parse number '" + value + "'");
                }
                continue;
            }
            std::istringstream row(line);
            double x = 0.0, y = 0.0;
            if (!(row >> x >> y))
                parse_error(path, no, "expected two numeric columns");
            std::string rest;
            if (row >> rest)
                parse_error(path, no, "trailing token '" + rest + "'");
            f->x[section].push_back(x);
            f->y[section].push_back(y);
        }
        if (!has_name || !has_z || !has_density)
            parse_error(path, no, "missing header key (name=, z_eff=, density=)");
        check_material(*f, z_eff, density);
        xs_material& m = f->view;
        m.name = f->name.c_str();
        m.z_eff = z_eff;
        m.density_ref = density;
        xs_table* t[6] = {&m.mu, &m.sigma_incoh, &m.sigma_coh, &m.sigma_pe, &m.s_factor, &m.f_factor};
        for (int k = 0; k < 6; ++k)
            *t[k] = xs_table{(int32_t)f->x[k].size(), f->x[k].data(), f->y[k].data()};
        *out = f.release();
    });
}

const xs_material* xs_material_file_get(const xs_material_file* f) { return f ? &f->view : nullptr; }
void xs_material_file_free(xs_material_file* f) { delete f; }

// --------------------------------------------------------------- spectrum
int xs_spectrum_file_load(const char* path, xs_spectrum_file** out)
{
    *out = nullptr;
    return run([&] {
        auto f = std::make_unique<xs_spectrum_file>();
        std::vector<double> cols[2];
        read_columns<2>(path, "spectrum", "two columns (keV, weight)", cols);
        f->e = std::move(cols[0]);
        f->w = std::move(cols[1]);
        f->view = xs_spectrum{(int32_t)f->e.size(), f->e.data(), f->w.data()};
        xsh::validate_spectrum(f->view); // REF spectrum.cpp:11-30
        *out = f.release();
    });
}

const xs_spectrum* xs_spectrum_file_get(const xs_spectrum_file* f) { return f ? &f->view : nullptr; }
void xs_spectrum_file_free(xs_spectrum_file* f) { delete f; }

// ------------------------------------------------------ detector response
int xs_response_file_load(const char* path_c, xs_response_file** out)
{
    *out = nullptr;
    return run([&] {
        const std::string path = path_c;
        auto f = std::make_unique<xs_response_file>();
        std::vector<double> cols[3];
        read_columns<3>(path, "detector response", "three columns (keV, dqe, deposit_keV)", cols);
        if (cols[0].empty())
            raise(path + ": empty detector response");
        // REF Table1D(e, ., "dqe") / ("deposit"): the abscissa must increase
        for (size_t i = 1; i < cols[0].size(); ++i)
            if (!(cols[0][i] > cols[0][i - 1]))
                raise("dqe: non-monotone abscissa");
        for (double v : cols[1])
            if (!(v >= 0.0 && v <= 1.0))
                raise("detector response: dqe outside [0,1]");
        for (size_t i = 0; i < cols[0].size(); ++i)
            if (cols[2][i] > cols[0][i] * (1.0 + 1e-12))
                raise("detector response: deposit exceeds incident energy");
        f->e = std::move(cols[0]);
        f->dqe = std::move(cols[1]);
        f->dep = std::move(cols[2]);
        const int32_t n = (int32_t)f->e.size();
        f->view = xs_response{xs_table{n, f->e.data(), f->dqe.data()}, xs_table{n, f->e.data(), f->dep.data()}};
        *out = f.release();
    });
}

const xs_response* xs_response_file_get(const xs_response_file* f) { return f ? &f->view : nullptr; }
void xs_response_file_free(xs_response_file* f) { delete f; }

} // extern "C"
