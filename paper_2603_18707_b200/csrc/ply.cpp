// ply.cpp — standard 3DGS checkpoint loader (load_ply, scene_io.cpp:53-199) into
// the SoA layout the device scene takes, so a real checkpoint runs through the
// same parity path as the synthetic scenes.
//
// Header rules, property lookup, the SH degree from the f_rest count and every
// error (type and message) follow the reference. The activations
// (sigmoid(opacity), exp(scale), normalized quaternion) are applied on the host
// in fp64 with the reference's expressions and the same libm, so the doubles
// handed to the device equal the reference's Splat3D fields bit for bit; the SH
// coefficients are float32 in the file and stay exact in the fp32 SH planes.
// The file is memory-mapped and decoded by all host threads.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "polysplat_b200.h"

namespace ps {
extern thread_local std::string g_free_error;
}

namespace {

struct PlyError {
    int status;
    std::string msg;
};

struct Prop {
    std::string name, type;
    size_t offset = 0, size = 0;
};

struct Element {
    std::string name;
    size_t count = 0, stride = 0;
    bool has_list = false;
    std::vector<Prop> props;
};

size_t type_size(const std::string& t) {
    if (t == "char" || t == "int8" || t == "uchar" || t == "uint8") return 1;
    if (t == "short" || t == "int16" || t == "ushort" || t == "uint16") return 2;
    if (t == "int" || t == "int32" || t == "uint" || t == "uint32") return 4;
    if (t == "float" || t == "float32") return 4;
    if (t == "double" || t == "float64") return 8;
    return 0;
}
bool is_f32(const std::string& t) { return t == "float" || t == "float32"; }

// The mapped file and the vertex layout the decoder needs.
struct PlyFile {
    const char* data = nullptr;
    size_t size = 0;
    int fd = -1;
    size_t data_off = 0, stride = 0;
    int64_t n = 0;
    int sh_degree = 0, per_channel = 0;
    size_t off_xyz[3], off_dc[3], off_op, off_scale[3], off_rot[4];
    std::vector<size_t> off_rest; // 3 * per_channel, channel-major

    ~PlyFile() {
        if (data) munmap(const_cast<char*>(data), size);
        if (fd >= 0) close(fd);
    }
};

void open_ply(const char* path, PlyFile& f) {
    if (!path) throw PlyError{PS_INVALID_ARGUMENT, "null path"};
    const std::string p(path);
    f.fd = open(path, O_RDONLY);
    struct stat st {};
    if (f.fd < 0 || fstat(f.fd, &st) != 0) throw PlyError{PS_IO_ERROR, "cannot open '" + p + "'"};
    f.size = static_cast<size_t>(st.st_size);
    if (f.size > 0) {
        void* m = mmap(nullptr, f.size, PROT_READ, MAP_PRIVATE, f.fd, 0);
        if (m == MAP_FAILED) throw PlyError{PS_IO_ERROR, "cannot open '" + p + "'"};
        f.data = static_cast<const char*>(m);
        madvise(m, f.size, MADV_SEQUENTIAL);
    }
    // header (scene_io.cpp:57-113)
    const std::string_view all(f.data ? f.data : "", f.size);
    const size_t he = all.find("end_header\n");
    if (he == std::string_view::npos) throw PlyError{PS_MALFORMED_HEADER, "missing end_header"};
    const size_t body = he + std::strlen("end_header\n");
    std::istringstream hs{std::string(all.substr(0, he))};
    std::string line;
    if (!std::getline(hs, line) || (line != "ply" && line != "ply\r"))
        throw PlyError{PS_MALFORMED_HEADER, "missing ply magic"};
    bool format_seen = false;
    std::vector<Element> els;
    while (std::getline(hs, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok.empty() || tok == "comment" || tok == "obj_info") continue;
        if (tok == "format") {
            std::string fmt, ver;
            ls >> fmt >> ver;
            if (fmt == "ascii" || fmt == "binary_big_endian")
                throw PlyError{PS_UNSUPPORTED_FORMAT, "only binary_little_endian PLY is supported"};
            if (fmt != "binary_little_endian" || ver != "1.0") throw PlyError{PS_MALFORMED_HEADER, "bad format line"};
            format_seen = true;
        } else if (tok == "element") {
            Element e;
            if (!(ls >> e.name >> e.count)) throw PlyError{PS_MALFORMED_HEADER, "bad element line"};
            els.push_back(e);
        } else if (tok == "property") {
            if (els.empty()) throw PlyError{PS_MALFORMED_HEADER, "property before element"};
            std::string type;
            ls >> type;
            Element& e = els.back();
            if (type == "list") {
                e.has_list = true;
                continue;
            }
            Prop pr;
            pr.type = type;
            pr.size = type_size(type);
            if (pr.size == 0) throw PlyError{PS_MALFORMED_HEADER, "unknown property type '" + type + "'"};
            if (!(ls >> pr.name)) throw PlyError{PS_MALFORMED_HEADER, "property without name"};
            pr.offset = e.stride;
            e.stride += pr.size;
            e.props.push_back(pr);
        } else {
            throw PlyError{PS_MALFORMED_HEADER, "unexpected header token '" + tok + "'"};
        }
    }
    if (!format_seen) throw PlyError{PS_MALFORMED_HEADER, "missing format line"};
    const Element* v = nullptr;
    size_t off = body;
    for (const Element& e : els) {
        if (e.name == "vertex") {
            v = &e;
            break;
        }
        if (e.has_list) throw PlyError{PS_UNSUPPORTED_FORMAT, "list properties before the vertex element"};
        off += e.stride * e.count;
    }
    if (!v) throw PlyError{PS_MISSING_PROPERTY, "no vertex element"};
    if (v->has_list) throw PlyError{PS_UNSUPPORTED_FORMAT, "vertex element has list properties"};
    std::map<std::string, const Prop*> props;
    for (const Prop& pr : v->props) props[pr.name] = &pr;
    auto req = [&](const std::string& name) -> size_t {
        auto it = props.find(name);
        if (it == props.end()) throw PlyError{PS_MISSING_PROPERTY, "missing property '" + name + "'"};
        if (!is_f32(it->second->type))
            throw PlyError{PS_UNSUPPORTED_FORMAT, "property '" + name + "' is not float32"};
        return it->second->offset;
    };
    // the reference's lookup order (scene_io.cpp:131-139)
    for (int k = 0; k < 3; ++k) f.off_xyz[k] = req(std::string(1, "xyz"[k]));
    for (int k = 0; k < 3; ++k) f.off_dc[k] = req("f_dc_" + std::to_string(k));
    f.off_op = req("opacity");
    for (int k = 0; k < 3; ++k) f.off_scale[k] = req("scale_" + std::to_string(k));
    for (int k = 0; k < 4; ++k) f.off_rot[k] = req("rot_" + std::to_string(k));
    int n_rest = 0;
    while (n_rest < 45) {
        auto it = props.find("f_rest_" + std::to_string(n_rest));
        if (it == props.end()) break;
        if (!is_f32(it->second->type)) throw PlyError{PS_UNSUPPORTED_FORMAT, "f_rest properties must be float32"};
        ++n_rest;
    }
    f.sh_degree = n_rest >= 45 ? 3 : n_rest >= 24 ? 2 : n_rest >= 9 ? 1 : 0;
    f.per_channel = n_rest >= 45 ? 15 : n_rest >= 24 ? 8 : n_rest >= 9 ? 3 : 0;
    for (int i = 0; i < 3 * f.per_channel; ++i) f.off_rest.push_back(props["f_rest_" + std::to_string(i)]->offset);
    if (f.size < off + v->stride * v->count) throw PlyError{PS_TRUNCATED_DATA, "vertex data shorter than declared"};
    f.data_off = off;
    f.stride = v->stride;
    f.n = static_cast<int64_t>(v->count);
}

inline double rd(const char* rec, size_t off) {
    float x;
    std::memcpy(&x, rec + off, 4);
    return static_cast<double>(x);
}

// Splat i's fields, with the reference's activations (scene_io.cpp:182-195).
struct Decoded {
    double mean[3], scale[3], rot[4], opacity;
    float sh[48]; // 16 coefficients x rgb, coefficient-major (Splat3D::sh order)
};

inline void decode(const PlyFile& f, int64_t i, Decoded& d) {
    const char* rec = f.data + f.data_off + static_cast<size_t>(i) * f.stride;
    for (int k = 0; k < 3; ++k) d.mean[k] = rd(rec, f.off_xyz[k]);
    d.opacity = 1.0 / (1.0 + std::exp(-rd(rec, f.off_op)));   // sigmoid
    for (int k = 0; k < 3; ++k) d.scale[k] = std::exp(rd(rec, f.off_scale[k]));
    const double w = rd(rec, f.off_rot[0]), x = rd(rec, f.off_rot[1]), y = rd(rec, f.off_rot[2]),
                 z = rd(rec, f.off_rot[3]);
    const double nrm = std::sqrt(w * w + x * x + y * y + z * z); // Quat::normalized (geometry.hpp:33-38)
    if (nrm < 1e-12) {
        d.rot[0] = 1.0; d.rot[1] = d.rot[2] = d.rot[3] = 0.0;
    } else {
        d.rot[0] = w / nrm; d.rot[1] = x / nrm; d.rot[2] = y / nrm; d.rot[3] = z / nrm;
    }
    std::memset(d.sh, 0, sizeof(d.sh));
    for (int c = 0; c < 3; ++c) d.sh[c] = static_cast<float>(rd(rec, f.off_dc[c]));
    for (int j = 0; j < f.per_channel; ++j)
        for (int c = 0; c < 3; ++c)
            d.sh[3 * (j + 1) + c] = static_cast<float>(rd(rec, f.off_rest[c * f.per_channel + j]));
}

template <typename Fn>
void parallel_for(int64_t n, Fn fn) {
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 65536));
    if (nt <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t a = t * chunk, b = std::min(n, a + chunk);
        if (a < b) th.emplace_back([=] { fn(a, b); });
    }
    for (auto& x : th) x.join();
}

int fail(const PlyError& e) {
    ps::g_free_error = e.msg;
    return e.status;
}

} // namespace

extern "C" {

int ps_ply_info(const char* path, int64_t* n_out, int* sh_degree) {
    try {
        PlyFile f;
        open_ply(path, f);
        if (n_out) *n_out = f.n;
        if (sh_degree) *sh_degree = f.sh_degree;
        return PS_OK;
    } catch (const PlyError& e) {
        return fail(e);
    }
}

int ps_ply_load_soa(const char* path, double* means, double* scales, double* rotations, double* opacities,
                    float* sh, int64_t capacity, int64_t* n_out, int* sh_degree) {
    try {
        PlyFile f;
        open_ply(path, f);
        if (n_out) *n_out = f.n;
        if (sh_degree) *sh_degree = f.sh_degree;
        if (f.n > capacity) throw PlyError{PS_INVALID_ARGUMENT, "capacity too small"};
        if (f.n > 0 && (!means || !scales || !rotations || !opacities || !sh))
            throw PlyError{PS_INVALID_ARGUMENT, "null output array"};
        parallel_for(f.n, [&](int64_t a, int64_t b) {
            Decoded d;
            for (int64_t i = a; i < b; ++i) {
                decode(f, i, d);
                std::memcpy(means + 3 * i, d.mean, sizeof(d.mean));
                std::memcpy(scales + 3 * i, d.scale, sizeof(d.scale));
                std::memcpy(rotations + 4 * i, d.rot, sizeof(d.rot));
                opacities[i] = d.opacity;
                std::memcpy(sh + 48 * i, d.sh, sizeof(d.sh));
            }
        });
        return PS_OK;
    } catch (const PlyError& e) {
        return fail(e);
    }
}

int ps_ply_load_splat3d(const char* path, double* splats, int64_t capacity, int64_t* n_out, int* sh_degree) {
    try {
        PlyFile f;
        open_ply(path, f);
        if (n_out) *n_out = f.n;
        if (sh_degree) *sh_degree = f.sh_degree;
        if (f.n > capacity) throw PlyError{PS_INVALID_ARGUMENT, "capacity too small"};
        if (f.n > 0 && !splats) throw PlyError{PS_INVALID_ARGUMENT, "null output array"};
        parallel_for(f.n, [&](int64_t a, int64_t b) {
            Decoded d;
            for (int64_t i = a; i < b; ++i) {
                decode(f, i, d);
                double* s = splats + PS_SPLAT3D_DOUBLES * i; // projection.hpp:13-19 layout
                std::memcpy(s, d.mean, sizeof(d.mean));
                std::memcpy(s + 3, d.scale, sizeof(d.scale));
                std::memcpy(s + 6, d.rot, sizeof(d.rot));
                s[10] = d.opacity;
                for (int k = 0; k < 48; ++k) s[11 + k] = d.sh[k];
            }
        });
        return PS_OK;
    } catch (const PlyError& e) {
        return fail(e);
    }
}

} // extern "C"
