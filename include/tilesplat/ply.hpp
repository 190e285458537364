// tilesplat/ply.hpp — ParameterStore <-> PLY and the
// training checkpoint ("PLY + config + optimizer-state
// sidecar").  Header-only host code; no device dependency.
//
// PLY layout is the de-facto 3DGS vertex element:
//   x y z  f_dc_0..2  f_rest_0..44  opacity  scale_0..2  rot_0..3
// with opacity a logit, scales logs and rot the raw quaternion (w x y z).
// f_rest is channel-major (f_rest_{c*15+k} = coefficient k of channel c) while
// the in-memory sh_rest is coefficient-major [N][15][3].
// The reader accepts ascii and binary_little_endian, any scalar property type,
// any property order and extra properties (e.g. nx ny nz); the writer emits the
// properties in the order above as float32.
//
// Optimizer sidecar (little-endian): "TSOPT001", int64 n, int64 step,
// m[59n], v[59n] (flat C-ABI layout), accum[n], vcount[n] as float32.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tilesplat.hpp"

namespace tilesplat {
namespace ply {

inline std::vector<std::string> property_names() {
    std::vector<std::string> p = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"};
    for (int i = 0; i < 45; ++i) p.push_back("f_rest_" + std::to_string(i));
    p.push_back("opacity");
    for (int i = 0; i < 3; ++i) p.push_back("scale_" + std::to_string(i));
    for (int i = 0; i < 4; ++i) p.push_back("rot_" + std::to_string(i));
    return p;  // 59 names
}

// row of 59 PLY values <-> Gaussian g of the store
inline void to_row(const ParameterStore& s, int64_t g, float* r) {
    for (int k = 0; k < 3; ++k) r[k] = s.means[3 * g + k];
    for (int k = 0; k < 3; ++k) r[3 + k] = s.sh_dc[3 * g + k];
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 15; ++k) r[6 + c * 15 + k] = s.sh_rest[45 * g + 3 * k + c];
    r[51] = s.opacity_logits[g];
    for (int k = 0; k < 3; ++k) r[52 + k] = s.log_scales[3 * g + k];
    for (int k = 0; k < 4; ++k) r[55 + k] = s.quaternions[4 * g + k];
}

inline void from_row(ParameterStore& s, int64_t g, const float* r) {
    for (int k = 0; k < 3; ++k) s.means[3 * g + k] = r[k];
    for (int k = 0; k < 3; ++k) s.sh_dc[3 * g + k] = r[3 + k];
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 15; ++k) s.sh_rest[45 * g + 3 * k + c] = r[6 + c * 15 + k];
    s.opacity_logits[g] = r[51];
    for (int k = 0; k < 3; ++k) s.log_scales[3 * g + k] = r[52 + k];
    for (int k = 0; k < 4; ++k) s.quaternions[4 * g + k] = r[55 + k];
}

inline void write(const std::string& path, const ParameterStore& s, bool binary = true) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw Error(TS_ERR_VALIDATION, "ply: cannot open " + path + " for writing");
    const int64_t n = s.size();
    f << "ply\nformat " << (binary ? "binary_little_endian" : "ascii") << " 1.0\n";
    f << "element vertex " << n << "\n";
    for (const auto& p : property_names()) f << "property float " << p << "\n";
    f << "end_header\n";
    std::vector<float> row(59);
    char buf[32];
    for (int64_t g = 0; g < n; ++g) {
        to_row(s, g, row.data());
        if (binary) {
            f.write(reinterpret_cast<const char*>(row.data()), 59 * sizeof(float));  // x86/ARM: little-endian
        } else {
            for (int k = 0; k < 59; ++k) {
                std::snprintf(buf, sizeof buf, "%.9g", double(row[k]));  // 9 digits round-trip fp32
                f << buf << (k == 58 ? '\n' : ' ');
            }
        }
    }
    if (!f) throw Error(TS_ERR_VALIDATION, "ply: write failed for " + path);
}

namespace detail {
inline int type_size(const std::string& t) {
    if (t == "char" || t == "uchar" || t == "int8" || t == "uint8") return 1;
    if (t == "short" || t == "ushort" || t == "int16" || t == "uint16") return 2;
    if (t == "int" || t == "uint" || t == "float" || t == "int32" || t == "uint32" || t == "float32") return 4;
    if (t == "double" || t == "float64") return 8;
    return 0;
}
inline double load(const std::string& t, const unsigned char* p) {
    if (t == "float" || t == "float32") { float v; std::memcpy(&v, p, 4); return v; }
    if (t == "double" || t == "float64") { double v; std::memcpy(&v, p, 8); return v; }
    if (t == "char" || t == "int8") return double(int8_t(p[0]));
    if (t == "uchar" || t == "uint8") return double(p[0]);
    if (t == "short" || t == "int16") { int16_t v; std::memcpy(&v, p, 2); return v; }
    if (t == "ushort" || t == "uint16") { uint16_t v; std::memcpy(&v, p, 2); return v; }
    if (t == "int" || t == "int32") { int32_t v; std::memcpy(&v, p, 4); return v; }
    uint32_t v; std::memcpy(&v, p, 4); return v;
}
}  // namespace detail

inline ParameterStore read(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error(TS_ERR_VALIDATION, "ply: cannot open " + path);
    std::string line;
    std::getline(f, line);
    if (line != "ply") throw Error(TS_ERR_VALIDATION, "ply: missing magic in " + path);
    bool binary = false, in_vertex = false, seen_vertex = false;
    int64_t n = -1;
    struct Prop { std::string type, name; };
    std::vector<Prop> props;
    while (std::getline(f, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        std::string w;
        ls >> w;
        if (w == "format") {
            std::string fmt;
            ls >> fmt;
            if (fmt == "binary_little_endian") binary = true;
            else if (fmt == "ascii") binary = false;
            else throw Error(TS_ERR_VALIDATION, "ply: unsupported format " + fmt);
        } else if (w == "element") {
            std::string name;
            int64_t cnt;
            ls >> name >> cnt;
            if (seen_vertex && !in_vertex) continue;
            in_vertex = name == "vertex";
            if (in_vertex) seen_vertex = true, n = cnt;
            else if (!seen_vertex) throw Error(TS_ERR_VALIDATION, "ply: element before vertex is unsupported");
        } else if (w == "property") {
            std::string type, name;
            ls >> type;
            ls >> name;
            if (in_vertex) {
                if (type == "list") throw Error(TS_ERR_VALIDATION, "ply: list properties in vertex are unsupported");
                if (!detail::type_size(type)) throw Error(TS_ERR_VALIDATION, "ply: bad type " + type);
                props.push_back({type, name});
            }
        } else if (w == "end_header") {
            break;
        }
    }
    if (n < 0) throw Error(TS_ERR_VALIDATION, "ply: no vertex element in " + path);
    const auto names = property_names();
    std::vector<int> col(59, -1);
    for (size_t j = 0; j < props.size(); ++j)
        for (int k = 0; k < 59; ++k)
            if (props[j].name == names[k]) col[k] = int(j);
    for (int k = 0; k < 59; ++k)
        if (col[k] < 0) throw Error(TS_ERR_VALIDATION, "ply: missing property " + names[k]);
    std::vector<int> off(props.size() + 1, 0);
    for (size_t j = 0; j < props.size(); ++j) off[j + 1] = off[j] + detail::type_size(props[j].type);
    ParameterStore s;
    s.resize(n);
    std::vector<unsigned char> raw(off.back());
    std::vector<double> vals(props.size());
    float row[59];
    for (int64_t g = 0; g < n; ++g) {
        if (binary) {
            if (!f.read(reinterpret_cast<char*>(raw.data()), std::streamsize(raw.size())))
                throw Error(TS_ERR_VALIDATION, "ply: truncated vertex data");
            for (size_t j = 0; j < props.size(); ++j) vals[j] = detail::load(props[j].type, raw.data() + off[j]);
        } else {
            for (size_t j = 0; j < props.size(); ++j)
                if (!(f >> vals[j])) throw Error(TS_ERR_VALIDATION, "ply: truncated ascii vertex data");
        }
        for (int k = 0; k < 59; ++k) row[k] = float(vals[col[k]]);
        from_row(s, g, row);
    }
    return s;
}

}  // namespace ply

// ---- checkpoint: <dir>/point_cloud.ply + <dir>/optimizer.bin (+ config.json by the trainer) ----
struct OptimizerState {
    int64_t step = 0;
    std::vector<float> m, v, accum, vcount;  // 59n, 59n, n, n
};

inline void write_optimizer_state(const std::string& path, int64_t n, const OptimizerState& st) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw Error(TS_ERR_VALIDATION, "checkpoint: cannot open " + path);
    f.write("TSOPT001", 8);
    f.write(reinterpret_cast<const char*>(&n), 8);
    f.write(reinterpret_cast<const char*>(&st.step), 8);
    f.write(reinterpret_cast<const char*>(st.m.data()), std::streamsize(59 * n * 4));
    f.write(reinterpret_cast<const char*>(st.v.data()), std::streamsize(59 * n * 4));
    f.write(reinterpret_cast<const char*>(st.accum.data()), std::streamsize(n * 4));
    f.write(reinterpret_cast<const char*>(st.vcount.data()), std::streamsize(n * 4));
    if (!f) throw Error(TS_ERR_VALIDATION, "checkpoint: write failed for " + path);
}

inline OptimizerState read_optimizer_state(const std::string& path, int64_t expect_n) {
    std::ifstream f(path, std::ios::binary);
    char magic[8];
    int64_t n = 0;
    OptimizerState st;
    if (!f.read(magic, 8) || std::memcmp(magic, "TSOPT001", 8) != 0)
        throw Error(TS_ERR_VALIDATION, "checkpoint: bad optimizer sidecar " + path);
    f.read(reinterpret_cast<char*>(&n), 8);
    f.read(reinterpret_cast<char*>(&st.step), 8);
    if (n != expect_n) throw Error(TS_ERR_VALIDATION, "checkpoint: sidecar N does not match the PLY");
    st.m.resize(59 * n), st.v.resize(59 * n), st.accum.resize(n), st.vcount.resize(n);
    f.read(reinterpret_cast<char*>(st.m.data()), std::streamsize(59 * n * 4));
    f.read(reinterpret_cast<char*>(st.v.data()), std::streamsize(59 * n * 4));
    f.read(reinterpret_cast<char*>(st.accum.data()), std::streamsize(n * 4));
    f.read(reinterpret_cast<char*>(st.vcount.data()), std::streamsize(n * 4));
    if (!f) throw Error(TS_ERR_VALIDATION, "checkpoint: truncated sidecar " + path);
    return st;
}

// Save / resume an Engine (params + Adam moments + densify statistics + step).
inline void save_checkpoint(Engine& e, const std::string& dir, int64_t step) {
    const int64_t n = e.size();
    ply::write(dir + "/point_cloud.ply", e.params(), true);
    OptimizerState st;
    st.step = step;
    st.m.resize(59 * n), st.v.resize(59 * n), st.accum.resize(n), st.vcount.resize(n);
    const ts_status r = ts_get_state(e.handle(), nullptr, st.m.data(), st.v.data(), st.accum.data(), st.vcount.data());
    if (r != TS_OK) throw Error(r, std::string("ts_get_state: ") + ts_last_error(e.handle()));
    write_optimizer_state(dir + "/optimizer.bin", n, st);
}

inline int64_t load_checkpoint(Engine& e, const std::string& dir) {
    const ParameterStore s = ply::read(dir + "/point_cloud.ply");
    const OptimizerState st = read_optimizer_state(dir + "/optimizer.bin", s.size());
    e.set_params(s);
    const ts_status r = ts_set_state(e.handle(), nullptr, st.m.data(), st.v.data(), st.accum.data(), st.vcount.data());
    if (r != TS_OK) throw Error(r, std::string("ts_set_state: ") + ts_last_error(e.handle()));
    return st.step;
}

}  // namespace tilesplat
