// io.cu — scene and camera files (scene_io.cpp:21-169), scene validation
// (scene.cpp:59-81) and scene_extent (scene.cpp:83-92).
//
// The PLY payload is the reference's: binary little-endian rows of 14
// doubles per splat (x y z scale_0..2 rot_0..3 opacity red green blue).
// The device path reads/writes that AoS block with one bulk copy and
// transposes to/from the resident group-major vector with a kernel; the
// validation that load_scene runs is a device pass that reports the first
// offending splat (lowest index, then the reference's check order).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>
#include <fstream>
#include <sstream>

#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

const char* const kPlyProperties[14] = {"x",     "y",     "z",     "scale_0", "scale_1",
                                        "scale_2", "rot_0", "rot_1", "rot_2",   "rot_3",
                                        "opacity", "red",   "green", "blue"};

[[noreturn]] void parse_fail(const std::string& path, int line, const std::string& what) {
    throw Error(SGTR_RUNTIME, path + ":" + std::to_string(line) + ": " + what);
}

// AoS row j of splat i  <->  group-major flat index (scene.hpp:37-52)
__host__ __device__ inline long long soa_index(long long K, long long i, int j) {
    if (j < 3) return 3 * i + j;
    if (j < 6) return 3 * K + 3 * i + (j - 3);
    if (j < 10) return 6 * K + 4 * i + (j - 6);
    if (j == 10) return 10 * K + i;
    return 11 * K + 3 * i + (j - 11);
}

__global__ void k_aos_to_soa(const double* __restrict__ aos, long long K,
                             double* __restrict__ soa) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 14 * K) return;
    const long long i = t / 14;
    const int j = (int)(t % 14);
    soa[soa_index(K, i, j)] = aos[t];
}

__global__ void k_soa_to_aos(const double* __restrict__ soa, long long K,
                             double* __restrict__ aos) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 14 * K) return;
    const long long i = t / 14;
    const int j = (int)(t % 14);
    aos[t] = soa[soa_index(K, i, j)];
}

// Scene::validate for one splat: 0 = valid, else the reference's first
// failing check (scene.cpp:60-80, in its order)
__host__ __device__ inline int validate_one(const double* x, long long K, long long i,
                                            const double* b) {
    for (int a = 0; a < 3; ++a) {
        const double mu = x[3 * i + a], s = x[3 * K + 3 * i + a], c = x[11 * K + 3 * i + a];
        if (!isfinite(mu) || !isfinite(s) || !isfinite(c)) return 1;
        if (s < b[0]) return 2;
        if (c < b[3] || c > b[4]) return 3;
    }
    const double* q = x + 6 * K + 4 * i;
    for (int a = 0; a < 4; ++a)
        if (!isfinite(q[a])) return 4;
    // Eigen's squaredNorm of a Vector4d reduces as (x^2 + z^2) + (y^2 + w^2)
    if ((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]) < 1e-24) return 5;
    const double al = x[10 * K + i];
    if (!isfinite(al) || al < b[1] || al > b[2]) return 6;
    return 0;
}

__global__ void k_validate(const double* __restrict__ x, long long K, double b0, double b1,
                           double b2, double b3, double b4, unsigned long long* first) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const double b[5] = {b0, b1, b2, b3, b4};
    const int code = validate_one(x, K, i, b);
    if (code) atomicMin(first, ((unsigned long long)i << 3) | (unsigned long long)code);
}

const char* validate_reason(int code) {
    switch (code) {
        case 1: return "non-finite parameter";
        case 2: return "scale below s_min";
        case 3: return "color out of range";
        case 4: return "non-finite quaternion";
        case 5: return "degenerate quaternion";
        default: return "opacity out of range";
    }
}

std::string num17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);  // ostream precision(17), default float
    return buf;
}

}  // namespace

PlyHeader ply_read_header(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(SGTR_RUNTIME, "load_scene: cannot open " + path);
    std::string line;
    int lineno = 0;
    auto next_line = [&]() {
        if (!std::getline(in, line)) parse_fail(path, lineno, "truncated header");
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
    };
    next_line();
    if (line != "ply") parse_fail(path, lineno, "not a PLY file");
    next_line();
    if (line != "format binary_little_endian 1.0")
        parse_fail(path, lineno, "unsupported format: " + line);
    long long count = -1;
    int props = 0;
    for (;;) {
        next_line();
        if (line == "end_header") break;
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok == "comment") continue;
        if (tok == "element") {
            std::string name;
            ls >> name >> count;
            if (name != "vertex" || count < 0)
                parse_fail(path, lineno, "expected 'element vertex <count>'");
            continue;
        }
        if (tok == "property") {
            std::string type, name;
            ls >> type >> name;
            if (type != "double") parse_fail(path, lineno, "property type must be double");
            if (props >= 14 || name != kPlyProperties[props])
                parse_fail(path, lineno, "unexpected property '" + name + "'");
            ++props;
            continue;
        }
        parse_fail(path, lineno, "unrecognized header line: " + line);
    }
    if (count < 0) parse_fail(path, lineno, "missing element vertex");
    if (props != 14)
        parse_fail(path, lineno, "expected 14 double properties, got " + std::to_string(props));
    PlyHeader h;
    h.count = count;
    h.data_offset = (long long)in.tellg();
    return h;
}

void ply_read_payload(const std::string& path, const PlyHeader& h, double* aos) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(SGTR_RUNTIME, "load_scene: cannot open " + path);
    in.seekg(h.data_offset);
    const long long bytes = 14LL * 8 * h.count;
    in.read(reinterpret_cast<char*>(aos), bytes);
    const long long got = in.gcount();
    if (got < bytes)
        throw Error(SGTR_RUNTIME,
                    path + ": truncated payload at element " + std::to_string(got / (14 * 8)));
}

void ply_write(const std::string& path, const double* aos, long long count) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(SGTR_RUNTIME, "save_scene: cannot open " + path);
    out << "ply\n"
        << "format binary_little_endian 1.0\n"
        << "comment splat-tr v1\n"
        << "element vertex " << count << "\n";
    for (const char* p : kPlyProperties) out << "property double " << p << "\n";
    out << "end_header\n";
    out.write(reinterpret_cast<const char*>(aos), 14LL * 8 * count);
    if (!out) throw Error(SGTR_RUNTIME, "save_scene: write failed for " + path);
}

void host_aos_to_soa(const double* aos, long long K, double* soa) {
    for (long long i = 0; i < K; ++i)
        for (int j = 0; j < 14; ++j) soa[soa_index(K, i, j)] = aos[14 * i + j];
}

void host_soa_to_aos(const double* soa, long long K, double* aos) {
    for (long long i = 0; i < K; ++i)
        for (int j = 0; j < 14; ++j) aos[14 * i + j] = soa[soa_index(K, i, j)];
}

void throw_invalid_splat(unsigned long long first) {
    if (first == ~0ull) return;
    throw Error(SGTR_RUNTIME, "splat " + std::to_string(first >> 3) + ": " +
                                  validate_reason((int)(first & 7)));
}

void host_validate(const double* x, long long K, const double b[5]) {
    for (long long i = 0; i < K; ++i) {
        const int code = validate_one(x, K, i, b);
        if (code) throw_invalid_splat(((unsigned long long)i << 3) | code);
    }
}

void launch_aos_to_soa(cudaStream_t st, const double* aos, long long K, double* soa) {
    if (K == 0) return;
    k_aos_to_soa<<<ceil_div(14 * K, 256), 256, 0, st>>>(aos, K, soa);
    SGTR_CUDA(cudaGetLastError());
}

void launch_soa_to_aos(cudaStream_t st, const double* soa, long long K, double* aos) {
    if (K == 0) return;
    k_soa_to_aos<<<ceil_div(14 * K, 256), 256, 0, st>>>(soa, K, aos);
    SGTR_CUDA(cudaGetLastError());
}

void launch_validate(cudaStream_t st, const double* x, long long K, const double b[5],
                     unsigned long long* first) {
    SGTR_CUDA(cudaMemsetAsync(first, 0xff, sizeof(*first), st));
    if (K == 0) return;
    k_validate<<<ceil_div(K, 256), 256, 0, st>>>(x, K, b[0], b[1], b[2], b[3], b[4], first);
    SGTR_CUDA(cudaGetLastError());
}

// save_cameras (scene_io.cpp:118-136)
void save_cameras(const std::string& path, const sgtr_camera* cams,
                  const char* const* names, int n) {
    std::ofstream out(path);
    if (!out) throw Error(SGTR_RUNTIME, "save_cameras: cannot open " + path);
    out << "# id fx fy cx cy width height qw qx qy qz tx ty tz image\n";
    for (int i = 0; i < n; ++i) {
        const sgtr_camera& c = cams[i];
        out << c.id << ' ' << num17(c.fx) << ' ' << num17(c.fy) << ' ' << num17(c.cx) << ' '
            << num17(c.cy) << ' ' << c.width << ' ' << c.height << ' ' << num17(c.q_wc[3])
            << ' ' << num17(c.q_wc[0]) << ' ' << num17(c.q_wc[1]) << ' ' << num17(c.q_wc[2])
            << ' ' << num17(c.t_wc[0]) << ' ' << num17(c.t_wc[1]) << ' ' << num17(c.t_wc[2])
            << ' ' << (names && names[i] ? names[i] : "") << "\n";
    }
    if (!out) throw Error(SGTR_RUNTIME, "save_cameras: write failed for " + path);
}

// load_cameras (scene_io.cpp:138-167) with load_images = false
std::vector<CameraLine> load_cameras(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error(SGTR_RUNTIME, "load_cameras: cannot open " + path);
    std::vector<CameraLine> cams;
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const auto hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        std::istringstream ls(line);
        CameraLine cl{};
        sgtr_camera& c = cl.cam;
        double qw, qx, qy, qz;
        if (!(ls >> c.id)) continue;  // blank line
        if (!(ls >> c.fx >> c.fy >> c.cx >> c.cy >> c.width >> c.height >> qw >> qx >> qy >>
              qz >> c.t_wc[0] >> c.t_wc[1] >> c.t_wc[2] >> cl.image_name))
            parse_fail(path, lineno, "malformed camera line");
        if (!(c.fx > 0.0) || !(c.fy > 0.0))
            parse_fail(path, lineno, "focal lengths must be positive");
        // Eigen Vector4d norm over (x, y, z, w): (x^2 + z^2) + (y^2 + w^2)
        const double nrm = std::sqrt((qx * qx + qz * qz) + (qy * qy + qw * qw));
        if (!(nrm > 1e-12)) parse_fail(path, lineno, "degenerate quaternion");
        c.q_wc[0] = qx / nrm;
        c.q_wc[1] = qy / nrm;
        c.q_wc[2] = qz / nrm;
        c.q_wc[3] = qw / nrm;
        cams.push_back(cl);
    }
    return cams;
}

// scene_extent (scene.cpp:83-92): largest camera-centre distance from the
// centroid, centre = -R^T t with R = R(q_wc)
double scene_extent(const sgtr_camera* cams, int n) {
    if (n < 2) return 1.0;
    std::vector<double> ctr(3LL * n);
    double cen[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) {
        double r[9];
        if (!quat_rot(cams[i].q_wc, r)) throw Error(SGTR_INVALID_ARGUMENT,
                                                        "quat_to_rotation: degenerate quaternion");
        for (int a = 0; a < 3; ++a) {
            ctr[3 * i + a] = -(r[a] * cams[i].t_wc[0] + r[3 + a] * cams[i].t_wc[1] +
                               r[6 + a] * cams[i].t_wc[2]);
            cen[a] += ctr[3 * i + a];
        }
    }
    for (double& v : cen) v /= static_cast<double>(n);
    double extent = 0.0;
    for (int i = 0; i < n; ++i) {
        const double dx = ctr[3 * i] - cen[0], dy = ctr[3 * i + 1] - cen[1],
                     dz = ctr[3 * i + 2] - cen[2];
        extent = std::max(extent, std::sqrt(dx * dx + dy * dy + dz * dz));
    }
    return extent > 0.0 ? extent : 1.0;
}

}  // namespace sgtr
