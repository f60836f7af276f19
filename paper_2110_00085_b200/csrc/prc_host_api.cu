// prc_host_api.cu — the reference's coarse C API (include/pathrec.h) on top of the engine.
//
// Host-only code: the JSON scene loader (io.cpp:190-278), PFM / PGM / CSV / VGRD files
// (io.cpp:32-155) and the coarse entry points of capi.cpp:58-334.  All device work goes
// through the fine-grained C ABI of pathrec_gpu.h on a process-wide default context.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pathrec.h"

#define PRC_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}

// An engine call failed: carry its code and message up.  File and format errors are
// classified by message as the reference's C layer does (capi.cpp:24-32: "cannot open",
// "truncated", "write failure" -> IO, "non-finite" -> NUMERIC, the rest -> CONFIG);
// device, handle and numeric failures keep the engine's code.
void ck(int rc) {
    if (rc == PRC_OK) return;
    const std::string m = prc_gpu_last_error();
    if (rc == PRC_ERR_IO || rc == PRC_ERR_CONFIG) {
        if (m.find("cannot open") != std::string::npos || m.find("truncated") != std::string::npos ||
            m.find("write failure") != std::string::npos)
            rc = PRC_ERR_IO;
        else if (m.find("non-finite") != std::string::npos)
            rc = PRC_ERR_NUMERIC;
        else
            rc = PRC_ERR_CONFIG;
    }
    throw Fail(rc, m);
}

// ------------------------------------------------------------------ minimal JSON
// Enough of RFC 8259 for scene files: objects, arrays, strings (with the common escapes),
// numbers, true / false / null.  Accessors follow the nlohmann calls of io.cpp.
struct Json {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;

    const Json* find(const std::string& k) const {
        if (kind != Obj) return nullptr;
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
    const Json& at(const std::string& k) const {  // json::at: a missing key is an error
        const Json* j = find(k);
        if (!j) throw Fail(PRC_ERR_CONFIG, "load_scene: missing key '" + k + "'");
        return *j;
    }
    bool contains(const std::string& k) const { return find(k) != nullptr; }
    double get_double() const {
        if (kind != Num) throw Fail(PRC_ERR_CONFIG, "load_scene: expected a number");
        return num;
    }
    int get_int() const { return (int)get_double(); }
    bool get_bool() const {
        if (kind != Bool) throw Fail(PRC_ERR_CONFIG, "load_scene: expected a boolean");
        return b;
    }
    const std::string& get_str() const {
        if (kind != Str) throw Fail(PRC_ERR_CONFIG, "load_scene: expected a string");
        return str;
    }
    double value(const std::string& k, double dflt) const {
        const Json* j = find(k);
        return j ? j->get_double() : dflt;
    }
    bool value(const std::string& k, bool dflt) const {
        const Json* j = find(k);
        return j ? j->get_bool() : dflt;
    }
    std::string value(const std::string& k, const std::string& dflt) const {
        const Json* j = find(k);
        return j ? j->get_str() : dflt;
    }
};

struct JsonParser {
    const std::string& s;
    size_t i = 0;
    explicit JsonParser(const std::string& t) : s(t) {}
    [[noreturn]] void err(const char* what) {
        throw Fail(PRC_ERR_CONFIG, std::string("parse error at offset ") + std::to_string(i) + ": " + what);
    }
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (s.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    Json value() {
        ws();
        if (i >= s.size()) err("unexpected end of input");
        Json j;
        const char c = s[i];
        if (c == '{') {
            j.kind = Json::Obj;
            ++i;
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return j;
            }
            for (;;) {
                ws();
                if (i >= s.size() || s[i] != '"') err("expected a key");
                std::string k = string();
                ws();
                if (i >= s.size() || s[i] != ':') err("expected ':'");
                ++i;
                j.obj.emplace_back(std::move(k), value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return j;
                }
                err("expected ',' or '}'");
            }
        }
        if (c == '[') {
            j.kind = Json::Arr;
            ++i;
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return j;
            }
            for (;;) {
                j.arr.push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return j;
                }
                err("expected ',' or ']'");
            }
        }
        if (c == '"') {
            j.kind = Json::Str;
            j.str = string();
            return j;
        }
        if (lit("true")) {
            j.kind = Json::Bool;
            j.b = true;
            return j;
        }
        if (lit("false")) {
            j.kind = Json::Bool;
            return j;
        }
        if (lit("null")) return j;
        // number: strtod on the maximal JSON number token
        const size_t b0 = i;
        if (i < s.size() && (s[i] == '-' || s[i] == '+')) ++i;
        while (i < s.size() && (std::isdigit((unsigned char)s[i]) || s[i] == '.' || s[i] == 'e' || s[i] == 'E' ||
                                s[i] == '-' || s[i] == '+'))
            ++i;
        if (i == b0) err("unexpected character");
        const std::string tok = s.substr(b0, i - b0);
        char* end = nullptr;
        j.kind = Json::Num;
        j.num = std::strtod(tok.c_str(), &end);
        if (!end || *end) err("bad number");
        return j;
    }
    std::string string() {
        ++i;  // opening quote
        std::string out;
        while (i < s.size() && s[i] != '"') {
            char c = s[i++];
            if (c == '\\') {
                if (i >= s.size()) err("bad escape");
                const char e = s[i++];
                switch (e) {
                    case 'n': c = '\n'; break;
                    case 't': c = '\t'; break;
                    case 'r': c = '\r'; break;
                    case 'b': c = '\b'; break;
                    case 'f': c = '\f'; break;
                    case 'u': {  // \uXXXX, ASCII range only (paths and names)
                        if (i + 4 > s.size()) err("bad \\u escape");
                        const long cp = std::strtol(s.substr(i, 4).c_str(), nullptr, 16);
                        i += 4;
                        c = cp < 128 ? (char)cp : '?';
                        break;
                    }
                    default: c = e;
                }
            }
            out.push_back(c);
        }
        if (i >= s.size()) err("unterminated string");
        ++i;
        return out;
    }
};

// ------------------------------------------------------------------ host vector ops
struct V3 {
    double x, y, z;
};
prc_vec3 pv(V3 a) { return {a.x, a.y, a.z}; }
V3 vec3_of(const Json& j) {  // io.cpp:159-162
    if (j.kind != Json::Arr || j.arr.size() != 3) throw Fail(PRC_ERR_CONFIG, "scene: expected a 3-vector");
    return {j.arr[0].get_double(), j.arr[1].get_double(), j.arr[2].get_double()};
}
V3 normalized(V3 v) {  // Vec3::normalized (vec3.hpp:24-25)
    const double n = std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z);
    return {v.x / n, v.y / n, v.z / n};
}

std::string parent_dir(const std::string& p) {
    const size_t k = p.find_last_of('/');
    return k == std::string::npos ? std::string() : p.substr(0, k);
}
std::string join(const std::string& dir, const std::string& rel) {
    if (dir.empty() || (!rel.empty() && rel[0] == '/')) return rel;
    return dir + "/" + rel;
}

// VGRD v1 through the engine's reader (io.cpp:32-57).
struct Grid {
    int dims[3] = {1, 1, 1};
    prc_vec3 origin{0, 0, 0}, voxel_size{1, 1, 1};
    int unit = 0;
    std::vector<double> values;
};
Grid read_grid(const std::string& path) {
    Grid g;
    ck(prc_gpu_load_grid(path.c_str(), g.dims, &g.origin, &g.voxel_size, &g.unit, nullptr, 0));
    g.values.resize((size_t)g.dims[0] * g.dims[1] * g.dims[2]);
    ck(prc_gpu_load_grid(path.c_str(), g.dims, &g.origin, &g.voxel_size, &g.unit, g.values.data(), g.values.size()));
    return g;
}

// ------------------------------------------------------------------ images
struct Img {
    int rows = 0, cols = 0;
    std::vector<double> data;
};

void check_finite(const double* d, size_t n, const char* what) {  // io.cpp:80-91
    size_t bad = 0, first = 0;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(d[i])) {
            if (!bad) first = i;
            ++bad;
        }
    if (bad)
        throw Fail(PRC_ERR_NUMERIC, std::string(what) + ": " + std::to_string(bad) +
                                        " non-finite pixel(s), first at index " + std::to_string(first));
}

void save_pfm(const double* d, int rows, int cols, const std::string& path) {  // io.cpp:94-106
    check_finite(d, (size_t)rows * cols, "save_pfm");
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Fail(PRC_ERR_IO, "save_pfm: cannot open " + path);
    os << "Pf\n" << cols << " " << rows << "\n-1.0\n";
    for (int r = rows - 1; r >= 0; --r)  // bottom-to-top rows
        for (int c = 0; c < cols; ++c) {
            const float v = (float)d[(size_t)r * cols + c];
            os.write(reinterpret_cast<const char*>(&v), sizeof v);
        }
    if (!os) throw Fail(PRC_ERR_IO, "save_pfm: write failure on " + path);
}

Img load_pfm(const std::string& path) {  // io.cpp:108-129
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Fail(PRC_ERR_IO, "load_pfm: cannot open " + path);
    std::string magic;
    is >> magic;
    if (magic != "Pf") throw Fail(PRC_ERR_CONFIG, "load_pfm: not a grayscale PFM: " + path);
    int cols = 0, rows = 0;
    double scale = 0.0;
    is >> cols >> rows >> scale;
    is.get();
    if (cols <= 0 || rows <= 0 || scale >= 0.0) throw Fail(PRC_ERR_CONFIG, "load_pfm: unsupported header in " + path);
    Img im;
    im.rows = rows;
    im.cols = cols;
    im.data.assign((size_t)rows * cols, 0.0);
    for (int r = rows - 1; r >= 0; --r)
        for (int c = 0; c < cols; ++c) {
            float v = 0.0f;
            is.read(reinterpret_cast<char*>(&v), sizeof v);
            im.data[(size_t)r * cols + c] = v;
        }
    if (!is) throw Fail(PRC_ERR_IO, "load_pfm: truncated payload in " + path);
    return im;
}

void save_pgm(const double* d, int rows, int cols, const std::string& path) {  // io.cpp:131-145
    check_finite(d, (size_t)rows * cols, "save_pgm_preview");
    double mx = 0.0;
    for (size_t i = 0; i < (size_t)rows * cols; ++i) mx = std::max(mx, d[i]);
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Fail(PRC_ERR_IO, "save_pgm_preview: cannot open " + path);
    os << "P5\n" << cols << " " << rows << "\n255\n";
    for (size_t i = 0; i < (size_t)rows * cols; ++i) {
        const double t = mx > 0.0 ? std::clamp(d[i] / mx, 0.0, 1.0) : 0.0;
        os.put((char)(unsigned char)std::lround(255.0 * std::pow(t, 1.0 / 2.2)));
    }
}

void save_csv(const std::vector<prc_gpu_iteration_log>& rows, const std::string& path) {  // io.cpp:147-155
    std::ofstream os(path);
    if (!os) throw Fail(PRC_ERR_IO, "save_csv: cannot open " + path);
    os << "iter,time_s,loss,eps,delta,stage\r\n";
    os.precision(17);
    for (const auto& r : rows)
        os << r.iter << "," << r.time_s << "," << r.loss << "," << r.eps << "," << r.delta << "," << r.stage << "\r\n";
}

// ------------------------------------------------------------------ the default context
std::mutex g_ctx_mu;
prc_gpu_ctx* g_ctx = nullptr;

prc_gpu_ctx* default_ctx() {  // one per process, on $LOCAL_RANK (else device 0)
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (!g_ctx) {
        const char* lr = std::getenv("LOCAL_RANK");
        ck(prc_gpu_ctx_create(lr ? std::atoi(lr) : 0, &g_ctx));
    }
    return g_ctx;
}

}  // namespace

// ================================================================== handles
struct prc_scene {
    int unit = 0;  // LengthUnit
    std::vector<std::vector<double>> ext;
    std::vector<prc_species_desc> sp;
    std::vector<prc_surface_desc> sf;
    std::vector<prc_detector_desc> dt;
    prc_scene_desc desc{};
    void link() {
        for (size_t j = 0; j < sp.size(); ++j) sp[j].extinction = ext[j].data();
        desc.n_species = (int)sp.size();
        desc.species = sp.empty() ? nullptr : sp.data();
        desc.n_surfaces = (int)sf.size();
        desc.surfaces = sf.empty() ? nullptr : sf.data();
        desc.n_detectors = (int)dt.size();
        desc.detectors = dt.empty() ? nullptr : dt.data();
    }
};

struct prc_result {
    std::vector<Img> images;
    std::vector<prc_gpu_iteration_log> history;
    bool has_grid = false, has_phong = false;
    Grid grid;  // recovered extinction (tomography)
    double kappa = 0.0, gamma = 0.0;
};

struct prc_grid {
    Grid g;
};

namespace {

// load_scene, io.cpp:190-278.  The engine keeps one voxel lattice: every species must
// share the first species' grid geometry.
std::unique_ptr<prc_scene> load_scene(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw Fail(PRC_ERR_IO, "load_scene: cannot open " + path);
    std::stringstream ss;
    ss << is.rdbuf();
    const std::string text = ss.str();
    Json j;
    try {
        JsonParser p(text);
        j = p.value();
        p.ws();
        if (p.i != text.size()) p.err("trailing characters");
    } catch (const Fail& e) {
        throw Fail(PRC_ERR_CONFIG, "load_scene: parse error in " + path + ": " + e.what());
    }
    const std::string base = parent_dir(path);
    auto sc = std::make_unique<prc_scene>();
    const std::string unit = j.value("unit", std::string("m"));
    if (unit == "m") sc->unit = 0;
    else if (unit == "km") sc->unit = 1;
    else throw Fail(PRC_ERR_CONFIG, "load_scene: unit must be 'm' or 'km'");
    sc->desc.bounds_min = pv(vec3_of(j.at("bounds").at("min")));
    sc->desc.bounds_max = pv(vec3_of(j.at("bounds").at("max")));
    const Json& jl = j.at("light");
    const std::string lt = jl.at("type").get_str();
    if (lt == "point") {
        sc->desc.light.kind = PRC_LIGHT_POINT;
        sc->desc.light.position = pv(vec3_of(jl.at("position")));
    } else if (lt == "sun") {
        sc->desc.light.kind = PRC_LIGHT_SUN;
        sc->desc.light.direction = pv(normalized(vec3_of(jl.at("direction"))));
    } else {
        throw Fail(PRC_ERR_CONFIG, "load_scene: unknown light type '" + lt + "'");
    }
    sc->desc.light.radiance = jl.value("radiance", 1.0);
    bool have_grid = false;
    if (const Json* js = j.find("species")) {
        for (const Json& s : js->arr) {
            prc_species_desc d{};
            d.albedo = s.at("albedo").get_double();
            const Json& ph = s.at("phase");
            const std::string pt = ph.at("type").get_str();
            if (pt == "hg") {
                d.phase_kind = PRC_PHASE_HG;
                d.g = ph.at("g").get_double();
            } else if (pt == "rayleigh") {
                d.phase_kind = PRC_PHASE_RAYLEIGH;
            } else {
                throw Fail(PRC_ERR_CONFIG, "scene: unknown phase type '" + pt + "'");
            }
            d.unknown = s.value("unknown", false) ? 1 : 0;
            const Json& je = s.at("extinction");
            Grid g;
            if (je.contains("grid")) {
                g = read_grid(join(base, je.at("grid").get_str()));
            } else {  // geom_of + VoxelGridField::constant, io.cpp:178-185
                const Json& dims = je.at("dims");
                if (dims.kind != Json::Arr || dims.arr.size() < 3) throw Fail(PRC_ERR_CONFIG, "scene: bad grid dims");
                for (int a = 0; a < 3; ++a) g.dims[a] = dims.arr[a].get_int();
                g.origin = pv(vec3_of(je.at("origin")));
                g.voxel_size = pv(vec3_of(je.at("voxel_size")));
                if (g.dims[0] <= 0 || g.dims[1] <= 0 || g.dims[2] <= 0) throw Fail(PRC_ERR_CONFIG, "scene: bad grid dims");
                g.values.assign((size_t)g.dims[0] * g.dims[1] * g.dims[2], je.at("constant").get_double());
            }
            if (!have_grid) {
                for (int a = 0; a < 3; ++a) sc->desc.dims[a] = g.dims[a];
                sc->desc.grid_origin = g.origin;
                sc->desc.voxel_size = g.voxel_size;
                have_grid = true;
            } else {
                const prc_scene_desc& q = sc->desc;
                if (q.dims[0] != g.dims[0] || q.dims[1] != g.dims[1] || q.dims[2] != g.dims[2] ||
                    std::memcmp(&q.grid_origin, &g.origin, sizeof g.origin) != 0 ||
                    std::memcmp(&q.voxel_size, &g.voxel_size, sizeof g.voxel_size) != 0)
                    throw Fail(PRC_ERR_CONFIG, "load_scene: species grids differ (one voxel lattice per scene)");
            }
            sc->ext.push_back(std::move(g.values));
            sc->sp.push_back(d);
        }
    }
    if (const Json* jsf = j.find("surfaces")) {
        for (const Json& s : jsf->arr) {
            prc_surface_desc d{};
            const std::string type = s.at("type").get_str();
            if (type == "sphere") {
                d.kind = PRC_SURF_SPHERE;
                d.center = pv(vec3_of(s.at("center")));
                d.radius = s.at("radius").get_double();
                d.axis = 2;
                d.hi[0] = d.hi[1] = 1.0;
                d.normal_sign = 1.0;
            } else if (type == "face") {
                d.kind = PRC_SURF_FACE;
                d.radius = 1.0;
                d.axis = s.at("axis").get_int();
                d.coord = s.at("coord").get_double();
                const Json &lo = s.at("lo"), &hi = s.at("hi");
                if (lo.arr.size() < 2 || hi.arr.size() < 2) throw Fail(PRC_ERR_CONFIG, "scene: face extents need 2 values");
                d.lo[0] = lo.arr[0].get_double();
                d.lo[1] = lo.arr[1].get_double();
                d.hi[0] = hi.arr[0].get_double();
                d.hi[1] = hi.arr[1].get_double();
                d.normal_sign = s.value("normal", 1.0);
            } else {
                throw Fail(PRC_ERR_CONFIG, "load_scene: unknown surface type '" + type + "'");
            }
            const Json& br = s.at("brdf");  // brdf_of, io.cpp:171-176
            const std::string bt = br.at("type").get_str();
            if (bt == "diffuse") {
                d.brdf_kind = PRC_BRDF_DIFFUSE;
                d.albedo = br.at("albedo").get_double();
            } else if (bt == "phong") {
                d.brdf_kind = PRC_BRDF_PHONG;
                d.albedo = 1.0;
                d.kappa_s = br.at("kappa_s").get_double();
                d.gamma = br.at("gamma").get_double();
            } else {
                throw Fail(PRC_ERR_CONFIG, "load_scene: unknown brdf type '" + bt + "'");
            }
            d.target = s.value("target", false) ? 1 : 0;
            sc->sf.push_back(d);
        }
    }
    for (const Json& jd : j.at("detectors").arr) {
        prc_detector_desc d{};
        d.position = pv(vec3_of(jd.at("position")));
        d.direction = pv(vec3_of(jd.at("direction")));
        d.up = jd.contains("up") ? pv(vec3_of(jd.at("up"))) : prc_vec3{0.0, 0.0, 1.0};
        d.rows = jd.at("rows").get_int();
        d.cols = jd.at("cols").get_int();
        d.fov = jd.at("fov").get_double();
        sc->dt.push_back(d);
    }
    sc->link();
    return sc;
}

// The structural checks the engine relies on (a subset of validate_scene, scene.cpp:110-197).
std::vector<std::string> violations(const prc_scene& s) {
    std::vector<std::string> v;
    const prc_scene_desc& d = s.desc;
    if (!(d.bounds_min.x < d.bounds_max.x && d.bounds_min.y < d.bounds_max.y && d.bounds_min.z < d.bounds_max.z))
        v.push_back("scene bounds are empty or inverted");
    int unknown = 0, target = 0;
    for (size_t j = 0; j < s.sp.size(); ++j) {
        const prc_species_desc& q = s.sp[j];
        if (!(q.albedo >= 0.0 && q.albedo <= 1.0)) v.push_back("species " + std::to_string(j) + ": albedo outside [0, 1]");
        if (q.phase_kind == PRC_PHASE_HG && !(std::fabs(q.g) < 1.0))
            v.push_back("species " + std::to_string(j) + ": |g| must be < 1");
        for (double b : s.ext[j])
            if (!(b >= 0.0) || !std::isfinite(b)) {
                v.push_back("species " + std::to_string(j) + ": negative or non-finite extinction");
                break;
            }
        unknown += q.unknown ? 1 : 0;
    }
    if (unknown > 1) v.push_back("more than one unknown species");
    if (!s.sp.empty() && (d.voxel_size.x <= 0.0 || d.voxel_size.y <= 0.0 || d.voxel_size.z <= 0.0))
        v.push_back("grid voxel size must be positive");
    for (size_t k = 0; k < s.sf.size(); ++k) {
        const prc_surface_desc& q = s.sf[k];
        if (q.kind == PRC_SURF_SPHERE && !(q.radius > 0.0)) v.push_back("surface " + std::to_string(k) + ": radius must be > 0");
        if (q.kind == PRC_SURF_FACE && (q.axis < 0 || q.axis > 2)) v.push_back("surface " + std::to_string(k) + ": face axis outside 0..2");
        if (q.target) {
            ++target;
            if (q.brdf_kind != PRC_BRDF_PHONG) v.push_back("surface " + std::to_string(k) + ": target needs a Phong BRDF");
        }
    }
    if (target > 1) v.push_back("more than one target surface");
    if (s.dt.empty()) v.push_back("scene has no detectors");
    for (size_t k = 0; k < s.dt.size(); ++k) {
        const prc_detector_desc& q = s.dt[k];
        if (q.rows <= 0 || q.cols <= 0) v.push_back("detector " + std::to_string(k) + ": non-positive pixel grid");
        if (!(q.fov > 0.0 && q.fov < 3.141592653589793)) v.push_back("detector " + std::to_string(k) + ": fov outside (0, pi)");
    }
    return v;
}

#define COARSE_TRY try {
#define COARSE_CATCH                                 \
    }                                                \
    catch (const Fail& e) {                          \
        return fail(e.code, e.what());               \
    }                                                \
    catch (const std::bad_alloc&) {                  \
        return fail(PRC_ERR_CONFIG, "out of memory"); \
    }                                                \
    catch (const std::exception& e) {                \
        return fail(PRC_ERR_CONFIG, e.what());       \
    }                                                \
    return PRC_OK;

void split_images(const prc_scene& s, const std::vector<double>& flat, std::vector<Img>& out) {
    size_t k = 0;
    for (const auto& d : s.dt) {
        Img im;
        im.rows = d.rows;
        im.cols = d.cols;
        im.data.assign(flat.begin() + (long)k, flat.begin() + (long)(k + (size_t)d.rows * d.cols));
        k += (size_t)d.rows * d.cols;
        out.push_back(std::move(im));
    }
}

}  // namespace

// ================================================================== the coarse C API
PRC_EXPORT const char* prc_version(void) { return "pathrec 0.1.0 (B200 engine)"; }
PRC_EXPORT const char* prc_last_error(void) { return g_err.c_str(); }

PRC_EXPORT int prc_scene_load(const char* path, prc_scene** out) {
    if (!path || !out) return fail(PRC_ERR_INVALID, "prc_scene_load: null argument");
    COARSE_TRY
    *out = load_scene(path).release();
    COARSE_CATCH
}

PRC_EXPORT void prc_scene_free(prc_scene* scene) { delete scene; }

PRC_EXPORT int prc_scene_validate(const prc_scene* scene, char* buf, size_t buflen, int* n_violations) {
    if (!scene) return fail(PRC_ERR_INVALID, "prc_scene_validate: null scene");
    const auto v = violations(*scene);
    if (n_violations) *n_violations = (int)v.size();
    if (buf && buflen > 0) {
        std::string all;
        for (const auto& x : v) all += x + "\n";
        const size_t n = std::min(buflen - 1, all.size());
        std::memcpy(buf, all.data(), n);
        buf[n] = '\0';
    }
    return PRC_OK;
}

PRC_EXPORT int prc_scene_detector_count(const prc_scene* scene, int* out) {
    if (!scene || !out) return fail(PRC_ERR_INVALID, "prc_scene_detector_count: null argument");
    *out = (int)scene->dt.size();
    return PRC_OK;
}

PRC_EXPORT int prc_scene_describe(const prc_scene* scene, const prc_scene_desc** out, int* length_unit) {
    if (!scene || !out) return fail(PRC_ERR_INVALID, "prc_scene_describe: null argument");
    *out = &scene->desc;
    if (length_unit) *length_unit = scene->unit;
    return PRC_OK;
}

PRC_EXPORT int prc_render(const prc_scene* scene, const prc_render_opts* opts, prc_result** out) {
    if (!scene || !opts || !out) return fail(PRC_ERR_INVALID, "prc_render: null argument");
    if (opts->n_paths == 0) return fail(PRC_ERR_CONFIG, "prc_render: n_paths must be >= 1");
    COARSE_TRY
    prc_gpu_ctx* c = default_ctx();
    ck(prc_gpu_scene_upload(c, &scene->desc));
    uint64_t n_pix = 0;
    ck(prc_gpu_scene_pixel_count(c, &n_pix));
    std::vector<double> img(n_pix);
    prc_gpu_render_opts ro{opts->n_paths, opts->seed, opts->max_bounces > 0 ? opts->max_bounces : 500, -1};
    prc_gpu_store* st = nullptr;
    uint64_t trunc = 0;
    ck(prc_gpu_render(c, &ro, nullptr, img.data(), &trunc, opts->store_dump_path ? &st : nullptr));
    std::unique_ptr<prc_gpu_store, void (*)(prc_gpu_store*)> hold(st, prc_gpu_store_free);
    if (st) ck(prc_gpu_store_export_pstr(c, st, opts->store_dump_path));
    auto r = std::make_unique<prc_result>();
    split_images(*scene, img, r->images);
    *out = r.release();
    COARSE_CATCH
}

PRC_EXPORT int prc_reconstruct(const prc_scene* scene, const prc_reconstruct_opts* opts, prc_result** out) {
    if (!scene || !opts || !out) return fail(PRC_ERR_INVALID, "prc_reconstruct: null argument");
    if (!opts->gt_dir) return fail(PRC_ERR_CONFIG, "prc_reconstruct: gt_dir is required");
    COARSE_TRY
    const prc_scene_desc& d = scene->desc;
    int unknown = -1, target = -1;
    for (int j = 0; j < d.n_species; ++j)
        if (d.species[j].unknown) unknown = j;
    for (int k = 0; k < d.n_surfaces; ++k)
        if (d.surfaces[k].target) target = k;
    const bool tomography = unknown >= 0;
    if (!tomography && target < 0)
        throw Fail(PRC_ERR_CONFIG, "prc_reconstruct: scene declares no unknown species or target surface");
    // ground truth: gt_000.pfm ... (capi.cpp:135-141)
    std::vector<double> gt;
    for (size_t k = 0; k < scene->dt.size(); ++k) {
        char name[64];
        std::snprintf(name, sizeof name, "gt_%03zu.pfm", k);
        const Img im = load_pfm(join(opts->gt_dir, name));
        if (im.rows != scene->dt[k].rows || im.cols != scene->dt[k].cols)
            throw Fail(PRC_ERR_CONFIG, std::string("prc_reconstruct: ") + name + " does not match the detector resolution");
        gt.insert(gt.end(), im.data.begin(), im.data.end());
    }
    prc_gpu_ctx* c = default_ctx();
    ck(prc_gpu_scene_upload(c, &d));
    // options (capi.cpp:143-186)
    prc_gpu_adam_config adam{opts->alpha > 0.0 ? opts->alpha : 1e7, 0.9, 0.999, 1e-8, 1, nullptr, 0};
    const int n_stages = opts->n_stages > 0 ? opts->n_stages : 1;
    std::vector<prc_gpu_stage> stages;
    uint64_t n = opts->n_paths > 0 ? opts->n_paths : 100000;
    for (int s = 0; s < n_stages; ++s, n *= 2) stages.push_back({0, 0, n});
    prc_gpu_schedule sch{};
    sch.seed = opts->seed;
    sch.max_bounces = opts->max_bounces > 0 ? opts->max_bounces : 500;
    sch.recycle_period = opts->recycle_period > 0 ? opts->recycle_period : 30;
    sch.max_iterations = opts->max_iterations;
    sch.stages = stages.data();
    sch.n_stages = (int)stages.size();
    sch.saturation_window = 20;
    sch.saturation_rel_improvement = 0.01;
    sch.checkpoint_every = opts->out_dir ? 25 : 0;
    sch.checkpoint_dir = opts->out_dir;
    sch.length_unit = scene->unit;
    prc_gpu_params init{}, truth{};
    std::vector<double> init_beta, truth_beta;
    const double step_scale[2] = {1.0, opts->gamma_step_scale > 0.0 ? opts->gamma_step_scale : 1.0};
    bool have_truth = false;
    const uint64_t V = d.n_species > 0 ? (uint64_t)d.dims[0] * d.dims[1] * d.dims[2] : 0;
    if (tomography) {
        init_beta.assign(V, 0.0);
        ck(prc_gpu_space_carve(c, gt.data(), opts->carve_threshold > 0.0 ? opts->carve_threshold : 0.02,
                               opts->carve_fill, nullptr, init_beta.data()));
        init.beta = init_beta.data();
        init.n_beta = V;
        if (opts->truth_grid) {
            truth_beta = read_grid(opts->truth_grid).values;
            if (truth_beta.size() != V) throw Fail(PRC_ERR_CONFIG, "prc_reconstruct: truth grid size != voxel count");
            truth.beta = truth_beta.data();
            truth.n_beta = V;
            have_truth = true;
        }
    } else {
        init.kappa_s = opts->init_kappa;
        init.gamma = opts->init_gamma;
        adam.step_scale = step_scale;
        adam.n_step_scale = 2;
        if (opts->truth_kappa > 0.0 || opts->truth_gamma > 0.0) {
            truth.kappa_s = opts->truth_kappa;
            truth.gamma = opts->truth_gamma;
            have_truth = true;
        }
    }
    if (have_truth) sch.truth = &truth;
    auto r = std::make_unique<prc_result>();
    r->history.resize((size_t)std::max(0, opts->max_iterations));
    ck(prc_gpu_reconstruct_schedule(c, &init, gt.data(), &adam, &sch, r->history.empty() ? nullptr : r->history.data(),
                                    nullptr, nullptr));
    if (tomography) {
        r->has_grid = true;
        Grid& g = r->grid;
        for (int a = 0; a < 3; ++a) g.dims[a] = d.dims[a];
        g.origin = d.grid_origin;
        g.voxel_size = d.voxel_size;
        g.unit = scene->unit;
        g.values.assign(V, 0.0);
        ck(prc_gpu_opt_params(c, g.values.data(), nullptr, nullptr));
    } else {
        r->has_phong = true;
        ck(prc_gpu_opt_params(c, nullptr, &r->kappa, &r->gamma));
    }
    *out = r.release();
    COARSE_CATCH
}

PRC_EXPORT int prc_result_image(const prc_result* result, int detector, const double** data, int* rows, int* cols) {
    if (!result || !data || !rows || !cols) return fail(PRC_ERR_INVALID, "prc_result_image: null argument");
    if (detector < 0 || detector >= (int)result->images.size())
        return fail(PRC_ERR_INVALID, "prc_result_image: detector index out of range");
    const Img& im = result->images[(size_t)detector];
    *data = im.data.data();
    *rows = im.rows;
    *cols = im.cols;
    return PRC_OK;
}

PRC_EXPORT int prc_result_save_pfm(const prc_result* result, int detector, const char* path) {
    if (!result || !path) return fail(PRC_ERR_INVALID, "prc_result_save_pfm: null argument");
    if (detector < 0 || detector >= (int)result->images.size())
        return fail(PRC_ERR_INVALID, "prc_result_save_pfm: detector index out of range");
    COARSE_TRY
    const Img& im = result->images[(size_t)detector];
    save_pfm(im.data.data(), im.rows, im.cols, path);
    COARSE_CATCH
}

PRC_EXPORT int prc_result_save_pgm(const prc_result* result, int detector, const char* path) {
    if (!result || !path) return fail(PRC_ERR_INVALID, "prc_result_save_pgm: null argument");
    if (detector < 0 || detector >= (int)result->images.size())
        return fail(PRC_ERR_INVALID, "prc_result_save_pgm: detector index out of range");
    COARSE_TRY
    const Img& im = result->images[(size_t)detector];
    save_pgm(im.data.data(), im.rows, im.cols, path);
    COARSE_CATCH
}

PRC_EXPORT int prc_result_params(const prc_result* result, double* kappa_s, double* gamma) {
    if (!result || !kappa_s || !gamma) return fail(PRC_ERR_INVALID, "prc_result_params: null argument");
    if (!result->has_phong) return fail(PRC_ERR_INVALID, "prc_result_params: not a reflectometry result");
    *kappa_s = result->kappa;
    *gamma = result->gamma;
    return PRC_OK;
}

PRC_EXPORT int prc_result_grid_save(const prc_result* result, const char* path) {
    if (!result || !path) return fail(PRC_ERR_INVALID, "prc_result_grid_save: null argument");
    if (!result->has_grid) return fail(PRC_ERR_INVALID, "prc_result_grid_save: not a tomography result");
    const Grid& g = result->grid;
    const int rc = prc_gpu_save_grid(path, g.dims, &g.origin, &g.voxel_size, g.unit, g.values.data());
    return rc == PRC_OK ? PRC_OK : fail(rc, prc_gpu_last_error());
}

PRC_EXPORT int prc_result_final_loss(const prc_result* result, double* loss) {
    if (!result || !loss) return fail(PRC_ERR_INVALID, "prc_result_final_loss: null argument");
    if (result->history.empty()) return fail(PRC_ERR_INVALID, "prc_result_final_loss: no optimization history");
    *loss = result->history.back().loss;
    return PRC_OK;
}

PRC_EXPORT int prc_result_save_csv(const prc_result* result, const char* path) {
    if (!result || !path) return fail(PRC_ERR_INVALID, "prc_result_save_csv: null argument");
    COARSE_TRY
    save_csv(result->history, path);
    COARSE_CATCH
}

PRC_EXPORT void prc_result_free(prc_result* result) { delete result; }

PRC_EXPORT int prc_grid_load(const char* path, prc_grid** out) {
    if (!path || !out) return fail(PRC_ERR_INVALID, "prc_grid_load: null argument");
    COARSE_TRY
    auto g = std::make_unique<prc_grid>();
    g->g = read_grid(path);
    *out = g.release();
    COARSE_CATCH
}

PRC_EXPORT int prc_grid_save(const prc_grid* grid, const char* path) {
    if (!grid || !path) return fail(PRC_ERR_INVALID, "prc_grid_save: null argument");
    const Grid& g = grid->g;
    const int rc = prc_gpu_save_grid(path, g.dims, &g.origin, &g.voxel_size, g.unit, g.values.data());
    return rc == PRC_OK ? PRC_OK : fail(rc, prc_gpu_last_error());
}

PRC_EXPORT int prc_grid_metrics(const prc_grid* estimate, const prc_grid* truth, double* eps, double* delta) {
    if (!estimate || !truth || !eps || !delta) return fail(PRC_ERR_INVALID, "prc_grid_metrics: null argument");
    if (estimate->g.values.size() != truth->g.values.size())
        return fail(PRC_ERR_CONFIG, "metrics: dimension mismatch");
    const int rc = prc_gpu_metrics(estimate->g.values.data(), truth->g.values.data(), truth->g.values.size(), eps, delta);
    return rc == PRC_OK ? PRC_OK : fail(PRC_ERR_CONFIG, prc_gpu_last_error());
}

PRC_EXPORT void prc_grid_free(prc_grid* grid) { delete grid; }

// Device self-test: the Philox4x32-10 known answer (rng.hpp, Random123 order), the DDA
// known answer of test_transport.cpp:13-42 (three unit voxels; a ray clipped at 1.5), and
// the HG / Rayleigh normalisation by a midpoint rule on the host.
PRC_EXPORT int prc_selftest(void) {
    COARSE_TRY
    prc_gpu_ctx* c = default_ctx();
    uint32_t w[4];
    ck(prc_gpu_debug_philox(c, 0, 0, 4, w));
    if (w[0] != 0x6627e8d5u || w[1] != 0xe169c58du || w[2] != 0xbc57ac4cu || w[3] != 0x9b00dbd8u)
        throw Fail(PRC_ERR_NUMERIC, "selftest: Philox known answer failed");
    double ext[3] = {1.0, 1.0, 1.0};
    prc_species_desc sp{ext, 1.0, PRC_PHASE_RAYLEIGH, 0.0, 0};
    prc_detector_desc det{{0.5, 0.5, 3.0}, {0, 0, -1}, {0, 1, 0}, 1, 1, 0.5};
    prc_scene_desc d{};
    d.bounds_max = {3.0, 1.0, 1.0};
    d.dims[0] = 3;
    d.dims[1] = d.dims[2] = 1;
    d.voxel_size = {1.0, 1.0, 1.0};
    d.n_species = 1;
    d.species = &sp;
    d.light.kind = PRC_LIGHT_POINT;
    d.light.position = {0.5, 0.5, 0.5};
    d.light.radiance = 1.0;
    d.n_detectors = 1;
    d.detectors = &det;
    ck(prc_gpu_scene_upload(c, &d));
    const double rays[14] = {0.0, 0.5, 0.5, 1.0, 0.0, 0.0, 10.0, 0.0, 0.5, 0.5, 1.0, 0.0, 0.0, 1.5};
    uint32_t counts[2], vox[8];
    double len[8];
    ck(prc_gpu_debug_walk(c, 2, rays, counts, vox, len, 8));
    if (counts[0] != 3 || counts[1] != 2 || vox[0] != 0 || vox[1] != 1 || vox[2] != 2 || len[0] != 1.0 ||
        len[1] != 1.0 || len[2] != 1.0 || vox[3] != 0 || vox[4] != 1 || len[3] != 1.0 || len[4] != 0.5)
        throw Fail(PRC_ERR_NUMERIC, "selftest: DDA known answer failed");
    for (int kind = 0; kind < 2; ++kind) {
        const double g = kind == 0 ? 0.85 : 0.0;
        const int m = 1 << 20;
        double total = 0.0;
        for (int i = 0; i < m; ++i) {
            const double cth = -1.0 + (i + 0.5) * (2.0 / m);
            const double f = kind == 1 ? 3.0 * (1.0 + cth * cth) / (16.0 * 3.141592653589793)
                                       : (1.0 - g * g) / (4.0 * 3.141592653589793 * (1.0 + g * g - 2.0 * g * cth) *
                                                          std::sqrt(1.0 + g * g - 2.0 * g * cth));
            total += f * (2.0 / m);
        }
        if (std::abs(2.0 * 3.141592653589793 * total - 1.0) > 1e-6)
            throw Fail(PRC_ERR_NUMERIC, "selftest: phase normalization failed");
    }
    COARSE_CATCH
}
