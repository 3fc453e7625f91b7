// host_common.cpp — GPU-free parts of the C ABI (validation, photon
// apportioning, Savitzky-Golay weights, scatter statistics finalize).
// Each function cites the reference code whose behaviour it reproduces.
#include "host_common.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <utility>

namespace xsh {

namespace {
thread_local std::string g_thread_error;
constexpr double kPi = 3.14159265358979323846;
} // namespace

void fail(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Error{code, buf};
}

int set_error(int code, const std::string& msg)
{
    g_thread_error = msg;
    return code;
}

const char* thread_error() { return g_thread_error.c_str(); }

void validate_sim_config(const xs_sim_config& c)
{
    if (c.photons_total < 1)
        fail(XS_E_RUNTIME, "sim config: photons_total must be >= 1");
    if (c.splitting < 1)
        fail(XS_E_RUNTIME, "sim config: splitting must be >= 1");
    if (!(c.roulette_survival > 0.0 && c.roulette_survival <= 1.0))
        fail(XS_E_RUNTIME, "sim config: roulette_survival must lie in (0,1]");
    if (c.roulette_wmin_rel < 0.0)
        fail(XS_E_RUNTIME, "sim config: roulette_wmin_rel must be >= 0");
    if (c.step_voxels < 1)
        fail(XS_E_RUNTIME, "sim config: step_voxels must be >= 1");
    if (c.max_interactions < 1)
        fail(XS_E_RUNTIME, "sim config: max_interactions must be >= 1");
}

void validate_spectrum(const xs_spectrum& s)
{
    if (s.n_bins <= 0)
        fail(XS_E_RUNTIME, "spectrum: no bins");
    double positive = 0.0;
    for (int i = 0; i < s.n_bins; ++i) {
        if (!std::isfinite(s.energy_kev[i]) || !std::isfinite(s.weight[i]))
            fail(XS_E_RUNTIME, "spectrum: non-finite entry");
        if (!(s.weight[i] >= 0.0))
            fail(XS_E_RUNTIME, "spectrum: negative weight");
        if (i > 0 && !(s.energy_kev[i] > s.energy_kev[i - 1]))
            fail(XS_E_RUNTIME, "spectrum: non-monotone abscissa");
        positive += s.weight[i];
    }
    if (!(positive > 0.0))
        fail(XS_E_RUNTIME, "spectrum: all weights zero");
    if (s.energy_kev[0] < 1.0 || s.energy_kev[s.n_bins - 1] > 1000.0)
        fail(XS_E_RUNTIME, "spectrum: energies must lie within [1 keV, 1 MeV]");
}

void validate_geometry(const xs_geometry& g)
{
    if (!(g.sod > 0.0 && g.sdd > g.sod))
        fail(XS_E_RUNTIME, "geometry: require 0 < sod < sdd");
    if (g.nu <= 0 || g.nv <= 0)
        fail(XS_E_RUNTIME, "geometry: detector pixel counts must be positive");
    if (!(g.pixel_pitch > 0.0))
        fail(XS_E_RUNTIME, "geometry: pixel pitch must be positive");
    if (g.n_angles <= 0 || !g.angles)
        fail(XS_E_RUNTIME, "geometry: no angles");
    for (int i = 0; i < g.n_angles; ++i) {
        if (g.angles[i] < 0.0 || g.angles[i] >= 2.0 * kPi)
            fail(XS_E_RUNTIME, "geometry: angles must lie in [0, 2pi)");
        if (i > 0 && !(g.angles[i] > g.angles[i - 1]))
            fail(XS_E_RUNTIME, "geometry: angles must be strictly increasing");
    }
}

std::vector<uint64_t> apportion(const xs_spectrum& spec, uint64_t photons_total)
{
    double w_total = 0.0;
    for (int i = 0; i < spec.n_bins; ++i)
        w_total += spec.weight[i];
    const std::size_t n = static_cast<std::size_t>(spec.n_bins);
    std::vector<uint64_t> counts(n, 0);
    std::vector<std::pair<double, std::size_t>> fractions;
    uint64_t assigned = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const double quota = photons_total * spec.weight[i] / w_total;
        counts[i] = static_cast<uint64_t>(quota);
        assigned += counts[i];
        fractions.emplace_back(quota - counts[i], i);
    }
    std::stable_sort(fractions.begin(), fractions.end(),
                     [](const auto& a, const auto& b) { return a.first > b.first; });
    for (std::size_t k = 0; assigned < photons_total && k < fractions.size(); ++k, ++assigned)
        ++counts[fractions[k].second];
    for (std::size_t i = 0; i < n; ++i)
        if (spec.weight[i] > 0.0 && counts[i] == 0)
            counts[i] = 1;
    return counts;
}

Frame frame_of(const xs_geometry& g, int angle_idx)
{
    Frame f;
    const double a = g.angles[angle_idx];
    const double r = g.sdd - g.sod;
    f.src[0] = g.sod * std::cos(a);
    f.src[1] = g.sod * std::sin(a);
    f.src[2] = 0.0;
    f.center[0] = -r * std::cos(a);
    f.center[1] = -r * std::sin(a);
    f.center[2] = 0.0;
    f.uaxis[0] = -std::sin(a);
    f.uaxis[1] = std::cos(a);
    f.uaxis[2] = 0.0;
    f.normal[0] = std::cos(a);
    f.normal[1] = std::sin(a);
    f.normal[2] = 0.0;
    return f;
}

namespace {
std::pair<int, bool> locate(const xs_table& t, double x)
{
    if (!(x >= t.x[0] && x <= t.x[t.n - 1]))
        fail(XS_E_OUT_OF_RANGE, "table: query %f outside [%f, %f]", x, t.x[0], t.x[t.n - 1]);
    int lo = 0, hi = t.n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (t.x[mid] <= x)
            lo = mid;
        else
            hi = mid;
    }
    if (x == t.x[lo])
        return {lo, true};
    if (x == t.x[hi])
        return {hi, true};
    return {lo, false};
}
} // namespace

double linear(const xs_table& t, double x)
{
    const auto [i, exact] = locate(t, x);
    if (exact)
        return t.y[i];
    const double u = (x - t.x[i]) / (t.x[i + 1] - t.x[i]);
    return t.y[i] + u * (t.y[i + 1] - t.y[i]);
}

double loglog(const xs_table& t, double x)
{
    const auto [i, exact] = locate(t, x);
    if (exact)
        return t.y[i];
    if (t.y[i] <= 0.0 || t.y[i + 1] <= 0.0) {
        const double u = (x - t.x[i]) / (t.x[i + 1] - t.x[i]);
        return t.y[i] + u * (t.y[i + 1] - t.y[i]);
    }
    const double u = (std::log(x) - std::log(t.x[i])) / (std::log(t.x[i + 1]) - std::log(t.x[i]));
    return std::exp(std::log(t.y[i]) + u * (std::log(t.y[i + 1]) - std::log(t.y[i])));
}

xsd::TabDesc pack_table(const xs_table& t, std::vector<double>& buf)
{
    xsd::TabDesc d;
    d.off = static_cast<int32_t>(buf.size());
    d.n = t.n;
    for (int i = 0; i < t.n; ++i)
        buf.push_back(t.x[i]);
    for (int i = 0; i < t.n; ++i)
        buf.push_back(t.y[i]);
    for (int i = 0; i < t.n; ++i)
        buf.push_back(std::log(t.x[i]));
    for (int i = 0; i < t.n; ++i)
        buf.push_back(t.y[i] > 0.0 ? std::log(t.y[i]) : 0.0);
    return d;
}

namespace {
void check_table(const char* mat, const char* tag, const xs_table& t)
{
    if (t.n <= 0 || !t.x || !t.y)
        fail(XS_E_RUNTIME, "material '%s': invariant violation: missing table [%s]", mat, tag);
    for (int i = 1; i < t.n; ++i)
        if (!(t.x[i] > t.x[i - 1]))
            fail(XS_E_RUNTIME, "material '%s': invariant violation: non-monotone abscissa in [%s]",
                 mat, tag);
}
} // namespace

void pack_materials(const xs_material* mats, int n, std::vector<double>& buf, xsd::MatDesc* out)
{
    for (int m = 0; m < n; ++m) {
        xsd::MatDesc& d = out[m];
        std::memset(&d, 0, sizeof d);
        const xs_material& mm = mats[m];
        if (m == 0 || mm.mu.n <= 0) { // vacuum / table-less sentinel
            d.has_tables = 0;
            continue;
        }
        const char* name = mm.name ? mm.name : "?";
        check_table(name, "mu", mm.mu);
        check_table(name, "incoherent", mm.sigma_incoh);
        check_table(name, "coherent", mm.sigma_coh);
        check_table(name, "photoelectric", mm.sigma_pe);
        check_table(name, "S", mm.s_factor);
        check_table(name, "F", mm.f_factor);
        d.has_tables = 1;
        d.z_eff = mm.z_eff;
        d.mu = pack_table(mm.mu, buf);
        d.incoh = pack_table(mm.sigma_incoh, buf);
        d.coh = pack_table(mm.sigma_coh, buf);
        d.pe = pack_table(mm.sigma_pe, buf);
        d.s = pack_table(mm.s_factor, buf);
        d.f = pack_table(mm.f_factor, buf);
        // F^2 dq^2 cumulative mass, REF material.cpp:107-125
        d.cdf_off = static_cast<int32_t>(buf.size());
        const double* q = mm.f_factor.x;
        const double* fv = mm.f_factor.y;
        double acc = 0.0;
        buf.push_back(0.0);
        for (int i = 1; i < mm.f_factor.n; ++i) {
            const double q0 = q[i - 1], q1 = q[i];
            const double a = fv[i - 1];
            const double b = (fv[i] - fv[i - 1]) / (q1 - q0);
            const double h = q1 - q0;
            const double c0 = a * a, c1 = 2.0 * a * b, c2 = b * b;
            const double integral = 2.0 * (c0 * q0 * h + (c0 + c1 * q0) * h * h / 2.0 +
                                           (c1 + c2 * q0) * h * h * h / 3.0 +
                                           c2 * h * h * h * h / 4.0);
            acc = acc + integral;
            buf.push_back(acc);
        }
    }
}

void validate_sg(int window, int polyorder)
{
    if (window < 5 || window % 2 == 0)
        fail(XS_E_RUNTIME, "sg filter: window must be odd and >= 5");
    if (polyorder < 0 || polyorder >= window)
        fail(XS_E_RUNTIME, "sg filter: polyorder must be < window");
}

std::vector<double> sg_kernel(int left, int right, int polyorder)
{
    const int n = left + right + 1;
    const int order = std::min(polyorder, n - 1);
    const int k = order + 1;
    std::vector<double> xtx(static_cast<std::size_t>(k) * k, 0.0);
    std::vector<double> powers(static_cast<std::size_t>(n) * k);
    for (int j = 0; j < n; ++j) {
        const double x = j - left;
        double p = 1.0;
        for (int m = 0; m < k; ++m) {
            powers[static_cast<std::size_t>(j) * k + m] = p;
            p *= x;
        }
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) {
            double s = 0.0;
            for (int j = 0; j < n; ++j)
                s += powers[static_cast<std::size_t>(j) * k + a] *
                     powers[static_cast<std::size_t>(j) * k + b];
            xtx[static_cast<std::size_t>(a) * k + b] = s;
        }
    // (X^T X) c = e0 by Gaussian elimination with partial pivoting
    std::vector<double> rhs(k, 0.0);
    rhs[0] = 1.0;
    for (int col = 0; col < k; ++col) {
        int pivot = col;
        for (int r = col + 1; r < k; ++r)
            if (std::abs(xtx[static_cast<std::size_t>(r) * k + col]) >
                std::abs(xtx[static_cast<std::size_t>(pivot) * k + col]))
                pivot = r;
        if (pivot != col) {
            for (int c = 0; c < k; ++c)
                std::swap(xtx[static_cast<std::size_t>(col) * k + c],
                          xtx[static_cast<std::size_t>(pivot) * k + c]);
            std::swap(rhs[col], rhs[pivot]);
        }
        const double diag = xtx[static_cast<std::size_t>(col) * k + col];
        if (diag == 0.0)
            fail(XS_E_RUNTIME, "sg_kernel: singular normal equations");
        for (int r = col + 1; r < k; ++r) {
            const double f = xtx[static_cast<std::size_t>(r) * k + col] / diag;
            for (int c = col; c < k; ++c)
                xtx[static_cast<std::size_t>(r) * k + c] -= f * xtx[static_cast<std::size_t>(col) * k + c];
            rhs[r] -= f * rhs[col];
        }
    }
    std::vector<double> coef(k);
    for (int r = k - 1; r >= 0; --r) {
        double s = rhs[r];
        for (int c = r + 1; c < k; ++c)
            s -= xtx[static_cast<std::size_t>(r) * k + c] * coef[c];
        coef[r] = s / xtx[static_cast<std::size_t>(r) * k + r];
    }
    std::vector<double> kernel(n);
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int m = 0; m < k; ++m)
            s += coef[m] * powers[static_cast<std::size_t>(j) * k + m];
        kernel[j] = s;
    }
    return kernel;
}

void finalize_stats(const xs_spectrum& spec, const std::vector<uint64_t>& counts,
                    uint64_t hist_begin, uint64_t hist_end, const uint64_t* bins,
                    const uint64_t* ledger, const xs_accum_units& units, xs_scatter_result* out)
{
    // per-bin history counts inside the covered range
    uint64_t base = 0;
    double total = 0.0, var_total = 0.0;
    uint64_t histories = 0;
    for (int b = 0; b < spec.n_bins; ++b) {
        const uint64_t lo = std::max(hist_begin, base);
        const uint64_t hi = std::min(hist_end, base + counts[b]);
        const uint64_t n = hi > lo ? hi - lo : 0;
        base += counts[b];
        const double sum_t = xs_dequantize(bins + 8 * b, units.log2_img);
        const double sum_t2 = xs_dequantize(bins + 8 * b + 3, 2 * units.log2_img);
        histories += n;
        total += sum_t;
        if (n > 1) {
            const double s2 = (sum_t2 - sum_t * sum_t / n) / (n - 1);
            var_total += n * std::max(0.0, s2);
        }
    }
    out->histories = histories;
    out->total = total;
    out->total_std_error = std::sqrt(var_total);
    double* led = &out->ledger.initial;
    for (int k = 0; k < 6; ++k)
        led[k] = xs_dequantize(ledger + 4 * k, units.log2_w);
}

} // namespace xsh

// ======================================================= extern "C" entry points
using namespace xsh;

namespace {
template <typename F>
int guard(F&& f)
{
    try {
        f();
        return XS_OK;
    } catch (const Error& e) {
        return set_error(e.code, e.msg);
    } catch (const std::exception& e) {
        return set_error(XS_E_RUNTIME, e.what());
    }
}
} // namespace

extern "C" {

const char* xs_version(void) { return "xscat-b200 0.1 (sm_100a)"; }
int xs_abi_version(void) { return XS_ABI_VERSION; }

void xs_sim_config_default(xs_sim_config* c)
{
    c->photons_total = 10000;
    c->splitting = 1;
    c->roulette_survival = 0.5;
    c->roulette_wmin_rel = 1e-3;
    c->step_voxels = 1;
    c->max_interactions = 50;
    c->seed = 0;
    c->track_variance = 0;
}

int xs_validate_sim_config(const xs_sim_config* c)
{
    return guard([&] { validate_sim_config(*c); });
}

int xs_apportion_photons(const xs_spectrum* spec, uint64_t photons_total, uint64_t* counts)
{
    return guard([&] {
        const auto c = apportion(*spec, photons_total);
        std::memcpy(counts, c.data(), c.size() * sizeof(uint64_t));
    });
}

int xs_history_count(const xs_spectrum* spec, uint64_t photons_total, uint64_t* n)
{
    return guard([&] {
        uint64_t s = 0;
        for (uint64_t c : apportion(*spec, photons_total))
            s += c;
        *n = s;
    });
}

// REF point_detector_score (transport.cpp:66-71)
double xs_point_detector_score(double response_factor, double p_dir, double weight,
                               double n_pixels, double d2, double tau)
{
    return response_factor * p_dir * weight * n_pixels / (2.0 * kPi * d2) * std::exp(-tau);
}

int xs_scatter_finalize_host(const xs_geometry* g, const xs_spectrum* spec,
                             const xs_sim_config* cfg, const uint64_t* accum, uint64_t hist_begin,
                             uint64_t hist_end, xs_scatter_result* out)
{
    return guard([&] {
        validate_sim_config(*cfg);
        validate_spectrum(*spec);
        validate_geometry(*g);
        const auto counts = apportion(*spec, cfg->photons_total);
        const xs_accum_units units = xs_accum_units_make(g, spec, counts.data());
        const xs_accum_layout L =
            xs_accum_layout_make(g->nu, g->nv, spec->n_bins, cfg->track_variance);
        finalize_stats(*spec, counts, hist_begin, hist_end, accum + L.off_bins,
                       accum + L.off_ledger, units, out);
        const double n = static_cast<double>(out->histories);
        for (uint64_t p = 0; p < L.n_pixels; ++p) {
            const double v = xs_dequantize(accum + L.off_image + 4 * p, units.log2_img);
            if (out->image)
                out->image[p] = v;
            if (cfg->track_variance && out->variance) {
                const double c2 = xs_dequantize(accum + L.off_variance + 4 * p, 2 * units.log2_img);
                out->variance[p] = std::max(0.0, c2 - v * v / n) * n / std::max(1.0, n - 1.0);
            }
        }
    });
}

int xs_validate_sg_spec(int32_t window, int32_t polyorder)
{
    return guard([&] { validate_sg(window, polyorder); });
}

// REF default_sg_spec (postprocess.cpp:19-26)
int xs_default_sg_spec(int32_t nu, int32_t nv, int32_t* window, int32_t* polyorder)
{
    const int smaller = std::min(nu, nv);
    int w = static_cast<int>(std::lround(15.0 * smaller / 576.0));
    w = std::max(5, w | 1);
    w = std::min(w, smaller % 2 ? smaller : smaller - 1);
    *window = w;
    *polyorder = 3;
    return XS_OK;
}

int xs_sg_kernel(int32_t left, int32_t right, int32_t polyorder, double* out)
{
    return guard([&] {
        const auto k = sg_kernel(left, right, polyorder);
        std::memcpy(out, k.data(), k.size() * sizeof(double));
    });
}

} // extern "C"
