// Replication-count sweeps and their CSV form (include/warpsim_b200.hpp; the reference's
// sweep.hpp:42-60 contract: rows per (mode, R) in canonical mode order, R ascending, the
// byte format of tests/golden/sweep_pi.golden).
//
// The CSV layout is one column table: each column knows its header name, how to print its
// field and how to read it back, and the header, emit_csv and parse_csv_string are all
// folds over that table. The sweep first lays out its points and then runs each one
// through run_model (GPU kernels via the C ABI), so the cycle columns are measured SM
// cycles of the sweep point's own launch.
#include <array>
#include <charconv>
#include <fstream>
#include <sstream>
#include <string_view>

#include "warpsim_b200.hpp"

namespace warpsim {
namespace {

[[noreturn]] void bad_field(std::size_t line, const char* kind, std::string_view text) {
    throw ParseError("csv line " + std::to_string(line) + ": bad " + kind + " '" + std::string(text) + "'");
}

template <class T>
T read_number(std::string_view text, std::size_t line, const char* kind) {
    T v{};
    const char* end = text.data() + text.size();
    const auto res = std::from_chars(text.data(), end, v);
    if (res.ec != std::errc{} || res.ptr != end) bad_field(line, kind, text);
    return v;
}

template <class T>
void write_number(std::string& out, T v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);  // doubles: shortest round trip
    out.append(buf, res.ptr);
}

// Names map to enumerators through the public lookups; a bad name is a parse error here.
template <class F>
auto read_name(std::string_view text, std::size_t line, F lookup) {
    try {
        return lookup(std::string(text));
    } catch (const DomainError& e) {
        throw ParseError("csv line " + std::to_string(line) + ": " + e.what());
    }
}

struct Column {
    const char* name;
    void (*put)(std::string&, const SweepRow&);
    void (*get)(SweepRow&, std::string_view, std::size_t);
};

#define WLP_INT_COLUMN(label, field)                                                                     \
    Column {                                                                                             \
        label, [](std::string& o, const SweepRow& r) { write_number(o, r.field); },                      \
            [](SweepRow& r, std::string_view t, std::size_t l) {                                          \
                r.field = read_number<decltype(SweepRow::field)>(t, l, "integer");                       \
            }                                                                                            \
    }
#define WLP_REAL_COLUMN(label, field)                                                                    \
    Column {                                                                                             \
        label, [](std::string& o, const SweepRow& r) { write_number(o, r.field); },                      \
            [](SweepRow& r, std::string_view t, std::size_t l) { r.field = read_number<double>(t, l, "real"); } \
    }

const std::array<Column, 11> kColumns = {
    WLP_INT_COLUMN("replications", replications),
    Column{"mode", [](std::string& o, const SweepRow& r) { o += mode_name(r.mode); },
           [](SweepRow& r, std::string_view t, std::size_t l) { r.mode = read_name(t, l, mode_from_name); }},
    Column{"model", [](std::string& o, const SweepRow& r) { o += model_name(r.model); },
           [](SweepRow& r, std::string_view t, std::size_t l) { r.model = read_name(t, l, model_from_name); }},
    WLP_INT_COLUMN("total_cycles", totalCycles),
    WLP_INT_COLUMN("mem_reads", memReads),
    WLP_INT_COLUMN("mem_writes", memWrites),
    WLP_INT_COLUMN("divergence_events", divergenceEvents),
    WLP_INT_COLUMN("waves", waves),
    WLP_REAL_COLUMN("mean", mean),
    WLP_REAL_COLUMN("ci_low", ciLow),
    WLP_REAL_COLUMN("ci_high", ciHigh),
};
#undef WLP_INT_COLUMN
#undef WLP_REAL_COLUMN

const std::string& header() {
    static const std::string h = [] {
        std::string s;
        for (const Column& c : kColumns) (s.empty() ? s : s += ',') += c.name;
        return s;
    }();
    return h;
}

// One data line: the fields between commas (an empty line yields one empty field).
std::vector<std::string_view> fields_of(std::string_view line) {
    std::vector<std::string_view> f;
    for (std::size_t at = 0;;) {
        const std::size_t comma = line.find(',', at);
        f.push_back(line.substr(at, comma == std::string_view::npos ? std::string_view::npos : comma - at));
        if (comma == std::string_view::npos) return f;
        at = comma + 1;
    }
}

// Mean and CI columns from the run's primary output: one replication has no interval.
void summarise(const std::vector<double>& primary, SweepRow& row) {
    if (primary.size() < 2) {
        row.mean = row.ciLow = row.ciHigh = primary.at(0);
        return;
    }
    const ConfidenceInterval ci = confidence_interval(primary);
    row.mean = ci.mean;
    row.ciLow = ci.low();
    row.ciHigh = ci.high();
}

}  // namespace

std::vector<SweepRow> run_sweep(const SweepSpec& spec, const DeviceProfile& prof) {
    if (spec.rMin < 1 || spec.rMax < spec.rMin) throw DomainError("sweep: need 1 <= rMin <= rMax");
    if (spec.rStep < 1) throw DomainError("sweep: rStep must be >= 1");
    if (spec.modes.empty()) throw DomainError("sweep: no execution modes selected");
    // the points, in the canonical order (modes Sequential, Tlp, Wlp; R ascending)
    std::vector<SweepRow> rows;
    for (const ExecutionMode mode : {ExecutionMode::Sequential, ExecutionMode::Tlp, ExecutionMode::Wlp}) {
        bool selected = false;
        for (const ExecutionMode m : spec.modes) selected |= m == mode;
        for (std::int64_t R = spec.rMin; selected && R <= spec.rMax; R += spec.rStep) {
            SweepRow row;
            row.replications = R;
            row.mode = mode;
            row.model = spec.model;
            rows.push_back(row);
        }
    }
    SimOptions opts;
    opts.irInterpreter = spec.irCounters;
    for (SweepRow& row : rows) {
        ModelParams params = spec.params;
        params.replications = row.replications;
        const ModelRun run = run_model(row.model, params, row.mode, prof, spec.masterSeed, spec.tlpBlockSize, opts);
        const SimReport& rep = run.report;  // measured on the GPU (cycles, counters, waves)
        row.totalCycles = rep.totalCycles;
        row.memReads = rep.memReads;
        row.memWrites = rep.memWrites;
        row.divergenceEvents = rep.divergenceEvents;
        row.waves = rep.wavesExecuted;
        summarise(run.primary, row);
    }
    return rows;
}

std::vector<std::int64_t> detect_steps(const std::vector<std::pair<std::int64_t, std::int64_t>>& curve) {
    std::vector<std::int64_t> rises;
    for (std::size_t i = 1; i < curve.size(); ++i) {
        const auto& [r_prev, c_prev] = curve[i - 1];
        const auto& [r, c] = curve[i];
        if (r <= r_prev) throw AnalysisError("step detection: curve not sorted by ascending R");
        if (c < c_prev)
            throw AnalysisError("step detection: cycles decreased at R=" + std::to_string(r) +
                                " — cost curves must be non-decreasing");
        if (c != c_prev) rises.push_back(r);
    }
    return rises;
}

std::vector<std::pair<std::int64_t, std::int64_t>> curve_of(const std::vector<SweepRow>& rows, ExecutionMode mode) {
    std::vector<std::pair<std::int64_t, std::int64_t>> points;
    for (const SweepRow& r : rows)
        if (r.mode == mode) points.emplace_back(r.replications, r.totalCycles);
    return points;
}

std::string csv_string(const std::vector<SweepRow>& rows) {
    std::string text = header() + '\n';
    for (const SweepRow& r : rows) {
        for (std::size_t k = 0; k < kColumns.size(); ++k) {
            if (k) text += ',';
            kColumns[k].put(text, r);
        }
        text += '\n';
    }
    return text;
}

void emit_csv(const std::vector<SweepRow>& rows, const std::string& path) {
    if (rows.empty()) throw DomainError("emit_csv: no rows");
    std::ofstream file(path);
    if (!file) throw Error("cannot write csv: " + path);
    file << csv_string(rows);
    if (!file.flush()) throw Error("write failed: " + path);
}

std::vector<SweepRow> parse_csv_string(const std::string& text) {
    std::vector<SweepRow> rows;
    std::size_t line_no = 0;
    for (std::size_t at = 0; at < text.size();) {
        const std::size_t nl = text.find('\n', at);
        std::string_view line(text.data() + at, (nl == std::string::npos ? text.size() : nl) - at);
        at = nl == std::string::npos ? text.size() : nl + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line_no == 1) {
            if (line != header()) throw ParseError("csv line 1: unexpected header");
            continue;
        }
        if (line.empty()) continue;
        const std::vector<std::string_view> f = fields_of(line);
        if (f.size() != kColumns.size())
            throw ParseError("csv line " + std::to_string(line_no) + ": expected " + std::to_string(kColumns.size()) +
                             " fields, got " + std::to_string(f.size()));
        SweepRow row;
        for (std::size_t k = 0; k < f.size(); ++k) kColumns[k].get(row, f[k], line_no);
        rows.push_back(row);
    }
    if (rows.empty()) throw ParseError("csv: no data rows");
    return rows;
}

std::vector<SweepRow> parse_csv(const std::string& path) {
    std::ifstream file(path, std::ios::binary);
    if (!file) throw Error("cannot open csv: " + path);
    std::ostringstream buf;
    buf << file.rdbuf();
    return parse_csv_string(buf.str());
}

}  // namespace warpsim
