// commands.cpp — the `lpsim` command layer on the B200 engine.
//
// Mirrors the reference's user surface so a user of `lpsim` can switch binaries:
//   * CLI           tools/lpsim_main.cpp:42-113  (subcommands, options, exit codes 2/3)
//   * commands      src/commands.cpp:46-216       (simulate / compare / cost / completeness /
//                                                  partition-plan, artifacts per output.formats)
//   * run config    src/run_config.cpp:85-247     (strict JSON schema, same error messages)
//   * artifacts     src/io.cpp:37-244             (LPLT latent dump, ledger / weight / cost CSV,
//                                                  summary JSON via nlohmann::json dump(2))
// Everything numeric comes from this library's C-ABI (include/lp_b200.h): plans, weights,
// cost model, completeness checker on the host; the denoising loop on the GPU engine.
// JSON is written with the same nlohmann/json (3.11.3) the reference uses, and CSV with
// default-formatted iostreams, so artifacts are byte-identical to the reference's.
//
// Host-only translation unit (g++); it reaches the device only through the C-ABI and
// cudaMemcpy of the engine's latent.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "lp_b200.h"

namespace lpb200 {
void set_last_error(const std::string& msg);  // lp_host.cpp (thread-local lp_last_error)
}

namespace {

using nlohmann::json;
namespace fs = std::filesystem;

struct CliError {
    int code;  // lp_status
    std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg) { throw CliError{code, msg}; }
[[noreturn]] void config_fail(const std::string& msg) { raise(LP_ERR_CONFIG, msg); }
void ck(int st) {
    if (st != LP_OK) raise(st, lp_last_error());
}
void cuda_ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(LP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

const char* kAxisNames[3] = {"temporal", "height", "width"};

struct Preset {
    std::string name;
    int64_t hidden;
    int dtype_bytes;
};
// builtin_presets (src/latent.cpp:197-206)
const std::vector<Preset>& presets() {
    static const std::vector<Preset> p = {{"wan21-like", 1536, 2}, {"fp32-small", 256, 4}};
    return p;
}

struct RunConfig {
    int64_t shape[4] = {1, 1, 1, 1};
    int dtype_bytes = 4;
    int64_t patch[3] = {1, 1, 1};
    int steps = 1;
    double eta = 0.0, guidance = 0.0;
    std::string kind = "box";
    int64_t radius[3] = {1, 1, 1};
    uint64_t seed = 0;
    int workers = 1;
    double r = 0.0;
    Preset preset;
    bool has_hybrid = false;
    int hybrid_m = 0;
    std::vector<int32_t> group_sizes;
    std::string dir = "out";
    bool out_json = true, out_csv = true, out_bin = true;
    int dit_layers = 30;  // extension: denoiser.kind "dit" (the engine's WAN2.1-1.3B-shaped DiT)
};

// ---- strict schema (src/run_config.cpp:85-233): same keys, checks and messages ----
void reject_unknown(const json& obj, const std::string& name, const std::set<std::string>& allowed) {
    for (const auto& it : obj.items())
        if (!allowed.count(it.key())) config_fail("unknown key '" + it.key() + "' in '" + name + "'");
}
const json& object_of(const json& doc, const std::string& name) {
    if (!doc.is_object()) config_fail("'" + name + "' must be a JSON object");
    return doc;
}
int64_t count_of(const json& obj, const std::string& name, const std::string& key, int64_t lo) {
    if (!obj.contains(key)) config_fail("'" + name + "' is missing required key '" + key + "'");
    const json& v = obj.at(key);
    if (!v.is_number_integer() && !v.is_number_unsigned()) config_fail("'" + name + "." + key + "' must be an integer");
    const int64_t x = v.get<int64_t>();
    if (x < lo) config_fail("'" + name + "." + key + "' must be >= " + std::to_string(lo));
    return x;
}
double number_of(const json& obj, const std::string& name, const std::string& key) {
    if (!obj.contains(key)) config_fail("'" + name + "' is missing required key '" + key + "'");
    const json& v = obj.at(key);
    if (!v.is_number()) config_fail("'" + name + "." + key + "' must be a number");
    return v.get<double>();
}

RunConfig parse_config(const json& doc) {
    object_of(doc, "config");
    reject_unknown(doc, "config", {"latent", "patch", "sampler", "denoiser", "cluster", "preset", "hybrid", "output"});
    RunConfig c;
    if (!doc.contains("latent")) config_fail("config is missing 'latent'");
    const json& lat = object_of(doc.at("latent"), "latent");
    reject_unknown(lat, "latent", {"C", "T", "H", "W", "dtype_bytes"});
    const char* dims[4] = {"C", "T", "H", "W"};
    for (int i = 0; i < 4; ++i) c.shape[i] = count_of(lat, "latent", dims[i], 1);
    if (lat.contains("dtype_bytes")) {
        const int64_t b = count_of(lat, "latent", "dtype_bytes", 2);
        if (b != 2 && b != 4 && b != 8) config_fail("'latent.dtype_bytes' must be 2, 4 or 8");
        c.dtype_bytes = static_cast<int>(b);
    }
    if (!doc.contains("patch")) config_fail("config is missing 'patch'");
    const json& pat = object_of(doc.at("patch"), "patch");
    reject_unknown(pat, "patch", {"p_T", "p_H", "p_W"});
    const char* pk[3] = {"p_T", "p_H", "p_W"};
    for (int a = 0; a < 3; ++a) c.patch[a] = count_of(pat, "patch", pk[a], 1);
    for (int a = 0; a < 3; ++a)
        if (c.shape[1 + a] < c.patch[a])
            config_fail(std::string("latent axis ") + kAxisNames[a] + " is smaller than its patch size");
    if (!doc.contains("sampler")) config_fail("config is missing 'sampler'");
    const json& smp = object_of(doc.at("sampler"), "sampler");
    reject_unknown(smp, "sampler", {"steps", "eta", "guidance_w"});
    c.steps = static_cast<int>(count_of(smp, "sampler", "steps", 1));
    c.eta = number_of(smp, "sampler", "eta");
    if (!(c.eta > 0.0)) config_fail("'sampler.eta' must be > 0");
    c.guidance = number_of(smp, "sampler", "guidance_w");
    if (!doc.contains("denoiser")) config_fail("config is missing 'denoiser'");
    const json& den = object_of(doc.at("denoiser"), "denoiser");
    // "dit" / "layers": extension of this engine (the reference has toy denoisers only)
    const bool is_dit = den.contains("kind") && den.at("kind").is_string() && den.at("kind").get<std::string>() == "dit";
    if (is_dit) reject_unknown(den, "denoiser", {"kind", "seed", "layers"});
    else reject_unknown(den, "denoiser", {"kind", "radius", "seed"});
    if (!den.contains("kind") || !den.at("kind").is_string()) config_fail("'denoiser.kind' must be a string");
    c.kind = den.at("kind").get<std::string>();
    if (c.kind != "box" && c.kind != "global" && c.kind != "identity" && c.kind != "dit")
        config_fail("'denoiser.kind' must be one of box, global, identity");
    if (den.contains("radius")) {
        const json& rad = den.at("radius");
        if (rad.is_number_integer() || rad.is_number_unsigned()) {
            const int64_t v = rad.get<int64_t>();
            if (v < 0) config_fail("'denoiser.radius' must be >= 0");
            c.radius[0] = c.radius[1] = c.radius[2] = v;
        } else if (rad.is_array() && rad.size() == 3) {
            for (size_t i = 0; i < 3; ++i) {
                if (!rad[i].is_number_integer() && !rad[i].is_number_unsigned())
                    config_fail("'denoiser.radius' entries must be integers");
                c.radius[i] = rad[i].get<int64_t>();
                if (c.radius[i] < 0) config_fail("'denoiser.radius' must be >= 0");
            }
        } else {
            config_fail("'denoiser.radius' must be an integer or an array of three integers");
        }
    }
    if (den.contains("seed")) {
        const json& s = den.at("seed");
        if (!s.is_number_unsigned() && !s.is_number_integer()) config_fail("'denoiser.seed' must be a non-negative integer");
        if (s.is_number_integer() && s.get<int64_t>() < 0) config_fail("'denoiser.seed' must be a non-negative integer");
        c.seed = s.get<uint64_t>();
    }
    if (is_dit && den.contains("layers")) c.dit_layers = static_cast<int>(count_of(den, "denoiser", "layers", 1));
    if (!doc.contains("cluster")) config_fail("config is missing 'cluster'");
    const json& clu = object_of(doc.at("cluster"), "cluster");
    reject_unknown(clu, "cluster", {"K", "r"});
    c.workers = static_cast<int>(count_of(clu, "cluster", "K", 1));
    c.r = number_of(clu, "cluster", "r");
    if (!(c.r >= 0.0 && c.r <= static_cast<double>(c.workers - 1))) config_fail("'cluster.r' must lie in [0, K-1]");
    std::string pname = "wan21-like";
    if (doc.contains("preset")) {
        if (!doc.at("preset").is_string()) config_fail("'preset' must be a string");
        pname = doc.at("preset").get<std::string>();
    }
    bool found = false;
    for (const Preset& p : presets())
        if (p.name == pname) c.preset = p, found = true;
    if (!found) config_fail("unknown preset '" + pname + "'");
    if (doc.contains("hybrid")) {
        const json& hy = object_of(doc.at("hybrid"), "hybrid");
        reject_unknown(hy, "hybrid", {"M", "group_sizes"});
        c.hybrid_m = static_cast<int>(count_of(hy, "hybrid", "M", 1));
        if (!hy.contains("group_sizes") || !hy.at("group_sizes").is_array())
            config_fail("'hybrid.group_sizes' must be an array");
        int total = 0;
        for (const json& v : hy.at("group_sizes")) {
            if (!v.is_number_integer() && !v.is_number_unsigned()) config_fail("'hybrid.group_sizes' entries must be integers");
            const int k = v.get<int>();
            if (k < 1) config_fail("'hybrid.group_sizes' entries must be >= 1");
            c.group_sizes.push_back(k);
            total += k;
        }
        if (static_cast<int>(c.group_sizes.size()) != c.hybrid_m) config_fail("'hybrid.M' does not match the number of group sizes");
        if (total != c.workers) config_fail("'hybrid.group_sizes' must sum to cluster.K");
        c.has_hybrid = true;
    }
    if (doc.contains("output")) {
        const json& out = object_of(doc.at("output"), "output");
        reject_unknown(out, "output", {"dir", "formats"});
        if (out.contains("dir")) {
            if (!out.at("dir").is_string()) config_fail("'output.dir' must be a string");
            c.dir = out.at("dir").get<std::string>();
        }
        if (out.contains("formats")) {
            if (!out.at("formats").is_array()) config_fail("'output.formats' must be an array");
            c.out_json = c.out_csv = c.out_bin = false;
            for (const json& v : out.at("formats")) {
                if (!v.is_string()) config_fail("'output.formats' entries must be strings");
                const std::string f = v.get<std::string>();
                if (f == "json") c.out_json = true;
                else if (f == "csv") c.out_csv = true;
                else if (f == "bin") c.out_bin = true;
                else config_fail("unknown output format '" + f + "'");
            }
        }
    }
    return c;
}

RunConfig load_config(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) raise(LP_ERR_CONFIG, "cannot open config file '" + path + "'");
    json doc;
    try {
        doc = json::parse(in);
    } catch (const json::exception& e) {
        raise(LP_ERR_CONFIG, std::string("config is not valid JSON: ") + e.what());
    }
    return parse_config(doc);
}

// ---- artifacts (src/io.cpp) ----
void write_text(const std::string& path, const std::string& s) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out || !out.write(s.data(), static_cast<std::streamsize>(s.size()))) raise(LP_ERR_IO, "cannot write '" + path + "'");
}
void write_json(const std::string& path, const json& doc) { write_text(path, doc.dump(2) + "\n"); }
std::string prepare_dir(const RunConfig& c) {
    std::error_code ec;
    fs::create_directories(c.dir, ec);
    if (ec) raise(LP_ERR_IO, "cannot create output directory '" + c.dir + "': " + ec.message());
    return c.dir;
}
std::string join(const std::string& d, const std::string& n) { return (fs::path(d) / n).string(); }

json config_echo(const RunConfig& c) {
    return {{"latent", {c.shape[0], c.shape[1], c.shape[2], c.shape[3]}},
            {"latent_dtype_bytes", c.dtype_bytes},
            {"patch", {c.patch[0], c.patch[1], c.patch[2]}},
            {"steps", c.steps},
            {"K", c.workers},
            {"r", c.r},
            {"denoiser", c.kind},
            {"seed", c.seed},
            {"preset", c.preset.name},
            {"preset_dtype_bytes", c.preset.dtype_bytes}};
}
json num_or_null(double v) { return std::isnan(v) ? json(nullptr) : json(v); }

double decode(const uint8_t* p, int db) {
    if (db == 2) {
        uint16_t h;
        std::memcpy(&h, p, 2);
        return lp_f16_decode(h);
    }
    if (db == 4) {
        float f;
        std::memcpy(&f, p, 4);
        return f;
    }
    double d;
    std::memcpy(&d, p, 8);
    return d;
}

// ---- the GPU engine behind run_lp (src/cluster.cpp:166-225) ----
struct Engine {
    lp_engine* e = nullptr;
    lp_dit* dit = nullptr;
    size_t bytes = 0;
    void* z = nullptr;
    Engine(const RunConfig& c, int workers, double r, const std::vector<double>& cond) {
        lp_engine_config ec{};
        for (int i = 0; i < 4; ++i) ec.shape[i] = c.shape[i];
        for (int a = 0; a < 3; ++a) ec.patch[a] = c.patch[a];  // K = 1: one entry = the whole latent
        ec.dtype_bytes = c.dtype_bytes;
        ec.workers = workers;
        ec.overlap_ratio = r;
        ec.total_steps = c.steps;
        ec.mode = LP_MODE_EXACT;
        ec.eta = c.eta;
        ec.guidance = c.guidance;
        ec.wire_bytes = c.preset.dtype_bytes;
        for (int a = 0; a < 3; ++a) ec.radius[a] = c.radius[a];
        ec.world = 1;
        ec.rank = 0;
        if (c.kind == "dit") {
            lp_dit_config dc;
            lp_dit_default_config(&dc);
            dc.num_layers = c.dit_layers;
            for (int a = 0; a < 3; ++a) dc.patch[a] = static_cast<int32_t>(c.patch[a]);
            dc.in_channels = static_cast<int32_t>(c.shape[0]);
            dc.t_scale = 1000.0 / c.steps;
            dc.seed = c.seed;
            ck(lp_dit_create(&dc, cond.data(), static_cast<int32_t>(cond.size()), &dit));
            ec.denoiser = -1;
            ec.dit = dit;
        } else {
            ec.denoiser = c.kind == "box" ? LP_TOY_BOX : (c.kind == "global" ? LP_TOY_GLOBAL : LP_TOY_IDENTITY);
            ec.t_coeff = c.kind == "identity" ? 0.0 : 0.01;  // make_*_denoiser defaults (include/lpsim/denoise.hpp)
            ec.cond_coeff = c.kind == "identity" ? 0.0 : 0.1;
        }
        ck(lp_engine_create(&ec, nullptr, cond.data(), static_cast<int32_t>(cond.size()), &e));
        ck(lp_engine_latent(e, &z));
        bytes = static_cast<size_t>(c.shape[0] * c.shape[1] * c.shape[2] * c.shape[3]) * c.dtype_bytes;
    }
    ~Engine() {
        if (e) lp_engine_destroy(e);
        if (dit) lp_dit_destroy(dit);
    }
    void upload(const std::vector<uint8_t>& bits) { cuda_ck(cudaMemcpy(z, bits.data(), bytes, cudaMemcpyHostToDevice), "upload"); }
    void run(int first, int count) {
        ck(lp_engine_run(e, first, count, nullptr));
        cuda_ck(cudaDeviceSynchronize(), "engine run");
        uint32_t flags = 0;
        ck(lp_device_flags(&flags, 1));
        if (flags & 1) raise(LP_ERR_NON_FINITE, "tensor element is not finite");
    }
    std::vector<uint8_t> download() const {
        std::vector<uint8_t> h(bytes);
        cuda_ck(cudaMemcpy(h.data(), z, bytes, cudaMemcpyDeviceToHost), "download");
        return h;
    }
};

// synthetic_inputs (src/run_config.cpp:258-301) as storage bits + cond values
std::vector<uint8_t> synthetic(const RunConfig& c, std::vector<double>& cond) {
    const size_t n = static_cast<size_t>(c.shape[0] * c.shape[1] * c.shape[2] * c.shape[3]);
    std::vector<double> v(n);
    cond.assign(8, 0.0);
    ck(lp_synthetic_inputs(c.shape, c.dtype_bytes, c.seed, v.data(), cond.data()));
    std::vector<uint8_t> bits(n * c.dtype_bytes);
    for (size_t i = 0; i < n; ++i) {
        if (c.dtype_bytes == 2) {
            const uint16_t h = lp_f16_encode(v[i]);
            std::memcpy(&bits[i * 2], &h, 2);
        } else if (c.dtype_bytes == 4) {
            const float f = static_cast<float>(v[i]);
            std::memcpy(&bits[i * 4], &f, 4);
        } else {
            std::memcpy(&bits[i * 8], &v[i], 8);
        }
    }
    return bits;
}

// CommLedger of run_lp (src/cluster.cpp:186-209): per step, per pass, scatter 1->k then
// (after the workers) gather k->1 for k >= 2, elements x preset dtype bytes.
struct Rec {
    int step;
    const char* pass;
    const char* kind;
    int src, dst;
    uint64_t bytes;
};
std::vector<Rec> ledger_records(const RunConfig& c) {
    std::vector<Rec> recs;
    for (int i = 1; i <= c.steps; ++i) {
        lp_plan plan;
        ck(lp_build_plan(c.shape, c.patch, i, c.workers, c.r, &plan));
        std::vector<int64_t> off(plan.n_entries + 1);
        ck(lp_plan_offsets(&plan, c.shape, off.data()));
        for (const char* kind : {"scatter", "gather"})
            for (const char* pass : {"cond", "uncond"})
                for (int k = 2; k <= plan.n_entries; ++k) {
                    const uint64_t el = static_cast<uint64_t>(off[k] - off[k - 1]);
                    const bool sc = kind[0] == 's';
                    recs.push_back({i, pass, kind, sc ? 1 : k, sc ? k : 1, el * static_cast<uint64_t>(c.preset.dtype_bytes)});
                }
    }
    return recs;
}

lp_cost_report_t cost_of(const RunConfig& c) {
    lp_cost_report_t r;
    ck(lp_cost_report(c.steps, c.workers, c.r, c.shape, c.patch, c.preset.hidden, c.preset.dtype_bytes,
                      c.has_hybrid ? c.hybrid_m : 0, c.has_hybrid ? c.group_sizes.data() : nullptr, &r));
    return r;
}

std::vector<uint8_t> dump_bytes(const RunConfig& c, const std::vector<uint8_t>& bits) {
    std::vector<uint8_t> buf(32);
    const uint32_t hdr[7] = {1u, static_cast<uint32_t>(c.dtype_bytes), static_cast<uint32_t>(c.shape[0]),
                             static_cast<uint32_t>(c.shape[1]), static_cast<uint32_t>(c.shape[2]),
                             static_cast<uint32_t>(c.shape[3]), 0u};
    std::memcpy(buf.data(), "LPLT", 4);
    std::memcpy(buf.data() + 4, hdr, sizeof(hdr));
    buf.insert(buf.end(), bits.begin(), bits.end());
    return buf;
}

json simulate(const RunConfig& c) {
    const std::string dir = prepare_dir(c);
    std::vector<double> cond;
    const std::vector<uint8_t> z0 = synthetic(c, cond);
    Engine eng(c, c.workers, c.r, cond);
    eng.upload(z0);
    eng.run(1, c.steps);
    const std::vector<uint8_t> zT = eng.download();
    const std::vector<Rec> recs = ledger_records(c);
    uint64_t total = 0;
    std::map<int, uint64_t> per_worker;
    for (const Rec& r : recs) {
        total += r.bytes;
        per_worker[r.src] += r.bytes;
        per_worker[r.dst] += r.bytes;
    }
    json pw = json::object();
    for (const auto& [w, b] : per_worker) pw[std::to_string(w)] = b;
    json s = {{"grand_total", total}, {"per_worker_totals", pw}};
    s["command"] = "simulate";
    s["config"] = config_echo(c);
    s["total_bytes"] = total;
    s["formula_check"] = total == cost_of(c).lp_exact_bytes;
    s["files"] = json::array();
    if (c.out_bin) {
        const std::vector<uint8_t> d = dump_bytes(c, zT);
        write_text(join(dir, "z0.bin"), std::string(d.begin(), d.end()));
        s["files"].push_back("z0.bin");
    }
    if (c.out_csv) {
        std::ostringstream os;
        os << "step,pass,kind,src,dst,bytes\n";
        for (const Rec& r : recs) os << r.step << ',' << r.pass << ',' << r.kind << ',' << r.src << ',' << r.dst << ',' << r.bytes << '\n';
        write_text(join(dir, "ledger.csv"), os.str());
        s["files"].push_back("ledger.csv");
    }
    if (c.out_json) {
        s["files"].push_back("summary.json");
        write_json(join(dir, "summary.json"), s);
    }
    return s;
}

json compare(const RunConfig& c) {
    const std::string dir = prepare_dir(c);
    std::vector<double> cond;
    const std::vector<uint8_t> z0 = synthetic(c, cond);
    Engine lp(c, c.workers, c.r, cond), central(c, 1, 0.0, cond);
    lp.upload(z0);
    central.upload(z0);
    const size_t n = lp.bytes / c.dtype_bytes;
    std::ostringstream diff;
    diff << "step,max_abs_diff,rms_diff\n";
    double fmax = 0.0, frms = 0.0;
    for (int i = 1; i <= c.steps; ++i) {
        lp.run(i, 1);
        central.run(i, 1);
        const std::vector<uint8_t> a = lp.download(), b = central.download();
        double m = 0.0, acc = 0.0;  // max_abs_diff / rms_diff (src/latent.cpp:173-195)
        for (size_t k = 0; k < n; ++k) {
            const double d = decode(&a[k * c.dtype_bytes], c.dtype_bytes) - decode(&b[k * c.dtype_bytes], c.dtype_bytes);
            m = std::max(m, std::abs(d));
            acc += d * d;
        }
        const double rms = n ? std::sqrt(acc / static_cast<double>(n)) : 0.0;
        diff << i << ',' << m << ',' << rms << '\n';
        fmax = m, frms = rms;
    }
    uint64_t lp_total = 0;
    for (const Rec& r : ledger_records(c)) lp_total += r.bytes;
    // run_nmp_emulation / run_pp_emulation(cfg.workers, ...) (src/cluster.cpp:229-280):
    // 2 passes x (K-1) boundaries x tokens x hidden per step, at the preset width
    const lp_cost_report_t cr = cost_of(c);
    const uint64_t emu = 2ull * static_cast<uint64_t>(c.steps) * static_cast<uint64_t>(c.workers - 1) * cr.activation_bytes;
    json s = {{"command", "compare"},
              {"config", config_echo(c)},
              {"final_max_abs_diff", fmax},
              {"final_rms_diff", frms},
              {"comm", {{"lp_total", lp_total}, {"nmp_total", emu}, {"pp_total", emu}}},
              {"files", json::array()}};
    if (c.out_csv) {
        write_text(join(dir, "diff.csv"), diff.str());
        s["files"].push_back("diff.csv");
    }
    if (c.out_json) {
        s["files"].push_back("compare.json");
        write_json(join(dir, "compare.json"), s);
    }
    return s;
}

json cost(const RunConfig& c) {
    const std::string dir = prepare_dir(c);
    const lp_cost_report_t r = cost_of(c);
    json s = {{"S_z", r.latent_bytes},
              {"S_H", r.activation_bytes},
              {"S_ext", r.ext_bytes_mean},
              {"gamma", r.gamma},
              {"gamma_per_axis", {r.gamma_per_axis[0], r.gamma_per_axis[1], r.gamma_per_axis[2]}},
              {"C_NMP", r.nmp_bytes},
              {"C_PP", r.pp_bytes},
              {"C_LP_exact", r.lp_exact_bytes},
              {"C_LP_approx", r.lp_approx_bytes},
              {"ratio_exact", num_or_null(r.ratio_exact)},
              {"ratio_approx", num_or_null(r.ratio_approx)},
              {"Sz_over_SH", r.latent_activation_ratio}};
    if (r.has_hybrid)
        s["hybrid"] = {{"C_inter", r.hybrid_inter_bytes},          {"C_intra_total", r.hybrid_intra_bytes},
                       {"C_hyb", r.hybrid_total_bytes},            {"ratio_vs_NMP", num_or_null(r.hybrid_ratio_vs_nmp)},
                       {"bound", num_or_null(r.hybrid_bound)},     {"within_bound", r.hybrid_within_bound != 0}};
    s["command"] = "cost";
    s["config"] = config_echo(c);
    if (c.out_csv) {
        std::ostringstream os;
        os << "T,K,r,C,D_T,D_H,D_W,p_T,p_H,p_W,preset,hidden_dim,dtype_bytes,S_z,S_H,gamma,"
              "C_NMP,C_PP,C_LP_exact,C_LP_approx,ratio_exact,ratio_approx\n";
        os << c.steps << ',' << c.workers << ',' << c.r << ',' << c.shape[0] << ',' << c.shape[1] << ',' << c.shape[2]
           << ',' << c.shape[3] << ',' << c.patch[0] << ',' << c.patch[1] << ',' << c.patch[2] << ',' << c.preset.name
           << ',' << c.preset.hidden << ',' << c.preset.dtype_bytes << ',' << r.latent_bytes << ','
           << r.activation_bytes << ',' << r.gamma << ',' << r.nmp_bytes << ',' << r.pp_bytes << ','
           << r.lp_exact_bytes << ',' << r.lp_approx_bytes << ',' << r.ratio_exact << ',' << r.ratio_approx << '\n';
        write_text(join(dir, "cost.csv"), os.str());
    }
    if (c.out_json) write_json(join(dir, "cost.json"), s);
    return s;
}

std::vector<int32_t> schedule_of(const std::string& name, int len) {
    std::vector<int32_t> s(static_cast<size_t>(len));
    for (int i = 1; i <= len; ++i) {
        if (name == "rotating") ck(lp_rotation_axis(i, &s[static_cast<size_t>(i - 1)]));
        else if (name == "temporal") s[static_cast<size_t>(i - 1)] = 0;
        else if (name == "height") s[static_cast<size_t>(i - 1)] = 1;
        else if (name == "width") s[static_cast<size_t>(i - 1)] = 2;
        else config_fail("unknown schedule '" + name + "'");
    }
    return s;
}

json completeness(const RunConfig& c, const std::string& sched_name, int max_steps) {
    const std::string dir = prepare_dir(c);
    int64_t grid[3];
    for (int a = 0; a < 3; ++a) grid[a] = c.shape[1 + a] / c.patch[a];  // patch_count (config checked extent >= patch)
    const std::vector<int32_t> sched = schedule_of(sched_name, max_steps);
    int32_t complete = 0, at = -1;
    int64_t worst[3];
    ck(lp_verify_n_complete(grid, c.workers, c.r, sched.data(), max_steps, max_steps, 0, &complete, &at, worst, nullptr));
    json names = json::array();
    for (int32_t a : sched) names.push_back(kAxisNames[a]);
    json s = {{"command", "completeness"},
              {"grid", {grid[0], grid[1], grid[2]}},
              {"K", c.workers},
              {"r", c.r},
              {"schedule", names},
              {"complete_at", complete ? json(at) : json(nullptr)},
              {"worst_position", {worst[0], worst[1], worst[2]}}};
    if (c.out_csv) {
        std::vector<int64_t> rows(5 * static_cast<size_t>(max_steps));
        std::vector<double> mean(static_cast<size_t>(max_steps));
        int32_t nr = 0;
        ck(lp_coverage_trace(grid, c.workers, c.r, sched.data(), max_steps, max_steps, 0, rows.data(), mean.data(), &nr));
        std::ostringstream os;
        os << "step,min_reached,mean_reached,max_reached,complete_positions,total_positions\n";
        for (int i = 0; i < nr; ++i)
            os << rows[5 * i] << ',' << rows[5 * i + 1] << ',' << mean[i] << ',' << rows[5 * i + 2] << ',' << rows[5 * i + 3]
               << ',' << rows[5 * i + 4] << '\n';
        write_text(join(dir, "coverage.csv"), os.str());
    }
    if (c.out_json) write_json(join(dir, "completeness.json"), s);
    return s;
}

json partition_plan(const RunConfig& c, int step) {
    const std::string dir = prepare_dir(c);
    lp_plan plan;
    ck(lp_build_plan(c.shape, c.patch, step, c.workers, c.r, &plan));
    json entries = json::array();
    for (int k = 0; k < plan.n_entries; ++k) {
        const lp_entry& e = plan.entries[k];
        entries.push_back({{"k", e.worker_id},
                           {"core", {e.core_begin, e.core_end}},
                           {"ext", {e.ext_begin, e.ext_end}},
                           {"latent", {e.latent_begin, e.latent_end}},
                           {"delta", {e.delta_start, e.delta_end}}});
    }
    json s = {{"axis", kAxisNames[plan.axis]},
              {"step", plan.step_index},
              {"L", plan.patches_per_core},
              {"O", plan.overlap_patches},
              {"entries", entries}};
    if (c.out_csv) {
        std::ostringstream os;
        os << "position,worker_id,weight\n";
        for (int k = 0; k < plan.n_entries; ++k) {
            const lp_entry& e = plan.entries[k];
            std::vector<double> w(static_cast<size_t>(e.latent_end - e.latent_begin));
            ck(lp_weight_profile(&plan, k, w.data()));
            for (size_t j = 0; j < w.size(); ++j)
                os << (e.latent_begin + static_cast<int64_t>(j)) << ',' << e.worker_id << ',' << w[j] << '\n';
        }
        write_text(join(dir, "weights.csv"), os.str());
    }
    if (c.out_json) write_json(join(dir, "plan.json"), s);
    return s;
}

void cli_warning(const char* msg, void*) { std::fprintf(stderr, "lpsim: warning: %s\n", msg); }

const char* kUsage =
    "Latent-partitioned diffusion serving simulator (B200 engine)\n"
    "Usage: lpsim_b200 SUBCOMMAND --config PATH [--out DIR] [--seed N] [--quiet] [--backend b200]\n"
    "Subcommands:\n"
    "  simulate        Run the multi-worker loop and meter every transfer\n"
    "  compare         Run the cluster and the single-context loop on one seed\n"
    "  cost            Evaluate the analytic communication models\n"
    "  completeness    Receptive-field coverage analysis [--schedule rotating|temporal|height|width] [--max-steps N]\n"
    "  partition-plan  Dump the partition of one denoising step [--step N]\n";

bool parse_int(const std::string& s, long long& v) {
    try {
        size_t pos = 0;
        v = std::stoll(s, &pos);
        return pos == s.size();
    } catch (...) {
        return false;
    }
}

}  // namespace

// The `lpsim` main (tools/lpsim_main.cpp:42-113): 0 ok, 2 usage / config error, 3 other errors.
extern "C" int lp_cli_main(int argc, const char* const* argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty() || args[0] == "-h" || args[0] == "--help") {
        std::fputs(kUsage, args.empty() ? stderr : stdout);
        return args.empty() ? 2 : 0;
    }
    const std::string cmd = args[0];
    static const std::set<std::string> cmds = {"simulate", "compare", "cost", "completeness", "partition-plan"};
    if (!cmds.count(cmd)) {
        std::fprintf(stderr, "lpsim: error: unknown subcommand '%s'\n%s", cmd.c_str(), kUsage);
        return 2;
    }
    std::string config, out, schedule = "rotating", backend = "b200";
    std::optional<uint64_t> seed;
    bool quiet = false;
    long long max_steps = 8, step = 1;
    for (size_t i = 1; i < args.size(); ++i) {
        const std::string& a = args[i];
        auto value = [&](std::string& dst) {
            if (i + 1 >= args.size()) {
                std::fprintf(stderr, "lpsim: error: %s requires a value\n", a.c_str());
                return false;
            }
            dst = args[++i];
            return true;
        };
        std::string v;
        if (a == "--quiet") quiet = true;
        else if (a == "--config") { if (!value(config)) return 2; }
        else if (a == "--out") { if (!value(out)) return 2; }
        else if (a == "--backend") {
            if (!value(backend)) return 2;
            if (backend != "b200") {
                std::fprintf(stderr, "lpsim: error: --backend: only 'b200' is built into this binary\n");
                return 2;
            }
        } else if (a == "--seed") {
            long long s;
            if (!value(v)) return 2;
            if (!parse_int(v, s) || s < 0) {
                std::fprintf(stderr, "lpsim: error: --seed: invalid value '%s'\n", v.c_str());
                return 2;
            }
            seed = static_cast<uint64_t>(s);
        } else if (a == "--schedule" && cmd == "completeness") {
            if (!value(schedule)) return 2;
            if (schedule != "rotating" && schedule != "temporal" && schedule != "height" && schedule != "width") {
                std::fprintf(stderr, "lpsim: error: --schedule: '%s' not in {rotating, temporal, height, width}\n", schedule.c_str());
                return 2;
            }
        } else if (a == "--max-steps" && cmd == "completeness") {
            if (!value(v)) return 2;
            if (!parse_int(v, max_steps) || max_steps < 1) {
                std::fprintf(stderr, "lpsim: error: --max-steps: value must be a positive number\n");
                return 2;
            }
        } else if (a == "--step" && cmd == "partition-plan") {
            if (!value(v)) return 2;
            if (!parse_int(v, step) || step < 1) {
                std::fprintf(stderr, "lpsim: error: --step: value must be a positive number\n");
                return 2;
            }
        } else if (a == "-h" || a == "--help") {
            std::fputs(kUsage, stdout);
            return 0;
        } else {
            std::fprintf(stderr, "lpsim: error: unexpected argument '%s'\n", a.c_str());
            return 2;
        }
    }
    if (config.empty()) {
        std::fprintf(stderr, "lpsim: error: --config is required\n");
        return 2;
    }
    lp_set_warning_handler(quiet ? nullptr : cli_warning, nullptr);
    try {
        RunConfig c = load_config(config);
        if (!out.empty()) c.dir = out;
        if (seed) c.seed = *seed;
        json s;
        if (cmd == "simulate") s = simulate(c);
        else if (cmd == "compare") s = compare(c);
        else if (cmd == "cost") s = cost(c);
        else if (cmd == "completeness") s = completeness(c, schedule, static_cast<int>(max_steps));
        else s = partition_plan(c, static_cast<int>(step));
        if (!quiet) std::printf("%s\n", s.dump(2).c_str());
        std::fflush(stdout);
        return 0;
    } catch (const CliError& e) {
        std::fprintf(stderr, "lpsim: error: %s\n", e.msg.c_str());
        return e.code == LP_ERR_CONFIG ? 2 : 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "lpsim: error: %s\n", e.what());
        return 3;
    }
}

// LPLT latent dump (src/io.cpp:37-139): 32-byte header ("LPLT", u32 version 1, u32
// dtype_bytes, u32 C/T/H/W, u32 0) + row-major payload at the storage width.
// `bits` are the storage-dtype bits of the latent (what the engine keeps on the device).
extern "C" int lp_latent_dump_write(const char* path, const void* bits, const int64_t shape[4], int32_t dtype_bytes) {
    try {
        if (dtype_bytes != 2 && dtype_bytes != 4 && dtype_bytes != 8)
            raise(LP_ERR_INVALID_ARGUMENT, "dtype_bytes must be 2, 4 or 8, got " + std::to_string(dtype_bytes));
        RunConfig c;
        for (int i = 0; i < 4; ++i) c.shape[i] = shape[i];
        c.dtype_bytes = dtype_bytes;
        const size_t n = static_cast<size_t>(shape[0] * shape[1] * shape[2] * shape[3]) * dtype_bytes;
        const uint8_t* p = static_cast<const uint8_t*>(bits);
        const std::vector<uint8_t> d = dump_bytes(c, std::vector<uint8_t>(p, p + n));
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out || !out.write(reinterpret_cast<const char*>(d.data()), static_cast<std::streamsize>(d.size())))
            raise(LP_ERR_IO, std::string("cannot write latent dump '") + path + "'");
        return LP_OK;
    } catch (const CliError& e) {
        lpb200::set_last_error(e.msg);
        return e.code;
    }
}

// Reads a dump; with bits == NULL only the header is parsed (shape / dtype / byte count).
// Errors as read_latent_dump: Io for unreadable / foreign / truncated files, InvalidArgument
// for a bad dtype, NonFinite for inf/NaN payload values (LatentTensor::from_doubles).
extern "C" int lp_latent_dump_read(const char* path, int64_t shape_out[4], int32_t* dtype_out, void* bits,
                                   int64_t capacity_bytes) {
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) raise(LP_ERR_IO, std::string("cannot open latent dump '") + path + "'");
        std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        if (buf.size() < 32 || std::memcmp(buf.data(), "LPLT", 4) != 0)
            raise(LP_ERR_IO, std::string("'") + path + "' is not a latent dump");
        uint32_t h[7];
        std::memcpy(h, buf.data() + 4, sizeof(h));
        if (h[0] != 1u) raise(LP_ERR_IO, "unsupported latent dump version");
        const int db = static_cast<int>(h[1]);
        if (db != 2 && db != 4 && db != 8) raise(LP_ERR_INVALID_ARGUMENT, "dtype_bytes must be 2, 4 or 8, got " + std::to_string(db));
        const size_t n = static_cast<size_t>(h[2]) * h[3] * h[4] * h[5];
        if (buf.size() != 32 + n * db) raise(LP_ERR_IO, "latent dump payload size mismatch");
        if (h[2] < 1 || h[3] < 1 || h[4] < 1 || h[5] < 1)
            raise(LP_ERR_INVALID_ARGUMENT, "shape extents must be >= 1, got (" + std::to_string(h[2]) + "," +
                                               std::to_string(h[3]) + "," + std::to_string(h[4]) + "," +
                                               std::to_string(h[5]) + ")");
        for (int i = 0; i < 4; ++i) shape_out[i] = h[2 + i];
        *dtype_out = db;
        if (!bits) return LP_OK;
        if (capacity_bytes < static_cast<int64_t>(n * db)) raise(LP_ERR_INVALID_ARGUMENT, "latent dump buffer too small");
        const uint8_t* p = reinterpret_cast<const uint8_t*>(buf.data()) + 32;
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(decode(p + i * db, db))) raise(LP_ERR_NON_FINITE, "tensor element is not finite");
        std::memcpy(bits, p, n * db);
        return LP_OK;
    } catch (const CliError& e) {
        lpb200::set_last_error(e.msg);
        return e.code;
    }
}
