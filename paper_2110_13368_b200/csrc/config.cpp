// XML simulation configuration: reader, strict schema, validation, canonical
// serialization, and the microenvironment / agents a config describes
// (config.hpp; the reference's schema config.hpp:75-91, semantics
// config.cpp:128-288 and 494-566).
#include "config.hpp"

#include <algorithm>
#include <array>
#include <cctype>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <set>
#include <sstream>

namespace biodiff_b200 {

namespace {

[[noreturn]] void bad_config(const std::string& msg) { throw config_error(msg); }

// ---------------------------------------------------------------------------
// XML reader: one document, one root element. Text is trimmed and inner
// whitespace runs collapse to a single space; comments, processing
// instructions and DOCTYPE are skipped; attributes are recorded only as
// "present" (the schema has none).

struct XmlElement {
    std::string tag;
    std::string text;
    bool has_attributes = false;
    std::vector<XmlElement> children;
};

class XmlDocument {
public:
    XmlDocument(const std::string& src, std::string where) : src_(src), where_(std::move(where)) {}

    XmlElement read_root()
    {
        skip_misc();
        if (at_end() || src_[pos_] != '<') fail("expected <");
        XmlElement root = read_element();
        skip_misc();
        if (!at_end()) fail("expected end of data");
        return root;
    }

private:
    const std::string& src_;
    std::string where_;
    std::size_t pos_ = 0;

    bool at_end() const { return pos_ >= src_.size(); }
    bool looking_at(const char* s) const { return src_.compare(pos_, std::char_traits<char>::length(s), s) == 0; }

    [[noreturn]] void fail(const std::string& what) const
    {
        const long line = 1 + std::count(src_.begin(), src_.begin() + static_cast<long>(std::min(pos_, src_.size())), '\n');
        bad_config("malformed XML" + where_ + " line " + format_int(line) + ": " + what);
    }

    void skip_space()
    {
        while (!at_end() && std::isspace(static_cast<unsigned char>(src_[pos_]))) ++pos_;
    }

    void skip_past(const char* terminator)
    {
        const std::size_t e = src_.find(terminator, pos_);
        if (e == std::string::npos) {
            pos_ = src_.size();
            fail("unexpected end of data");
        }
        pos_ = e + std::char_traits<char>::length(terminator);
    }

    void skip_misc()
    {
        for (;;) {
            skip_space();
            if (looking_at("<!--")) skip_past("-->");
            else if (looking_at("<?")) skip_past("?>");
            else if (looking_at("<!DOCTYPE")) skip_past(">");
            else return;
        }
    }

    std::string read_name()
    {
        const std::size_t b = pos_;
        while (!at_end()) {
            const char c = src_[pos_];
            if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.' || c == ':')) break;
            ++pos_;
        }
        if (pos_ == b) fail("expected element name");
        return src_.substr(b, pos_ - b);
    }

    static void append_decoded(std::string& out, const std::string& raw)
    {
        for (std::size_t i = 0; i < raw.size(); ++i) {
            const std::size_t semi = raw[i] == '&' ? raw.find(';', i) : std::string::npos;
            if (semi == std::string::npos) {
                out += raw[i];
                continue;
            }
            const std::string e = raw.substr(i + 1, semi - i - 1);
            static const std::map<std::string, char> named = {
                {"lt", '<'}, {"gt", '>'}, {"amp", '&'}, {"quot", '"'}, {"apos", '\''}};
            if (auto it = named.find(e); it != named.end()) {
                out += it->second;
            } else if (e.size() > 1 && e[0] == '#') {
                const bool hex = e[1] == 'x' || e[1] == 'X';
                const std::string digits = e.substr(hex ? 2 : 1);
                const bool ok = !digits.empty() && std::all_of(digits.begin(), digits.end(), [&](char ch) {
                    return hex ? std::isxdigit(static_cast<unsigned char>(ch)) != 0
                               : std::isdigit(static_cast<unsigned char>(ch)) != 0;
                });
                if (!ok || digits.size() > 6) bad_config("malformed XML: invalid character reference &" + e + ";");
                out += static_cast<char>(std::stoul(digits, nullptr, hex ? 16 : 10));
            } else {
                out += raw.substr(i, semi - i + 1);
            }
            i = semi;
        }
    }

    static std::string collapse(const std::string& t)
    {
        std::string out;
        bool gap = false;
        for (char c : t) {
            if (std::isspace(static_cast<unsigned char>(c))) {
                gap = !out.empty();
                continue;
            }
            if (gap) out += ' ';
            gap = false;
            out += c;
        }
        return out;
    }

    XmlElement read_element()
    {
        ++pos_; // '<'
        XmlElement el;
        el.tag = read_name();
        for (;;) { // attributes, then '>' or '/>'
            skip_space();
            if (at_end()) fail("unexpected end of data");
            if (looking_at("/>")) {
                pos_ += 2;
                return el;
            }
            if (src_[pos_] == '>') {
                ++pos_;
                break;
            }
            read_name();
            skip_space();
            if (at_end() || src_[pos_] != '=') fail("expected =");
            ++pos_;
            skip_space();
            if (at_end() || (src_[pos_] != '"' && src_[pos_] != '\'')) fail("expected ' or \"");
            const char quote = src_[pos_++];
            skip_past(std::string(1, quote).c_str());
            el.has_attributes = true;
        }
        std::string raw;
        for (;;) { // content
            if (at_end()) fail("unexpected end of data");
            if (looking_at("</")) {
                pos_ += 2;
                if (read_name() != el.tag) fail("invalid closing tag name");
                skip_space();
                if (at_end() || src_[pos_] != '>') fail("expected >");
                ++pos_;
                break;
            }
            if (looking_at("<!--")) {
                skip_past("-->");
            } else if (looking_at("<![CDATA[")) {
                const std::size_t b = pos_ + 9;
                skip_past("]]>");
                raw += src_.substr(b, pos_ - 3 - b);
            } else if (looking_at("<?")) {
                skip_past("?>");
            } else if (src_[pos_] == '<') {
                el.children.push_back(read_element());
            } else {
                const std::size_t e = src_.find('<', pos_);
                if (e == std::string::npos) {
                    pos_ = src_.size();
                    fail("unexpected end of data");
                }
                append_decoded(raw, src_.substr(pos_, e - pos_));
                pos_ = e;
            }
        }
        el.text = collapse(raw);
        return el;
    }
};

// ---------------------------------------------------------------------------
// Strict schema: every child of an element must be claimed by name (at most
// once, except the repeated ones), elements carry no attributes.

class Claim {
public:
    Claim(const XmlElement& el, std::string path) : el_(el), path_(std::move(path))
    {
        if (el.has_attributes) bad_config("element " + path_ + " carries attributes; this schema uses none");
        for (const auto& c : el.children) ++count_[c.tag];
    }

    bool present(const std::string& key) const { return count_.count(key) != 0; }

    const XmlElement* single(const std::string& key)
    {
        auto it = count_.find(key);
        if (it == count_.end()) return nullptr;
        if (it->second > 1) bad_config("element " + path_ + "." + key + " appears more than once");
        claimed_.insert(key);
        for (const auto& c : el_.children)
            if (c.tag == key) return &c;
        return nullptr;
    }

    std::vector<const XmlElement*> every(const std::string& key)
    {
        claimed_.insert(key);
        std::vector<const XmlElement*> out;
        for (const auto& c : el_.children)
            if (c.tag == key) out.push_back(&c);
        return out;
    }

    std::optional<std::string> text(const std::string& key)
    {
        const XmlElement* c = single(key);
        if (!c) return std::nullopt;
        return trim(c->text);
    }

    template <class T>
    void number(const std::string& key, T& into)
    {
        if (auto t = text(key)) {
            const std::string where = path_ + "." + key;
            try {
                if constexpr (std::is_floating_point_v<T>) into = parse_double(*t, where);
                else into = static_cast<T>(parse_int(*t, where));
            } catch (const std::invalid_argument&) {
                bad_config("element " + where + " holds '" + *t + "', expected " +
                           (std::is_floating_point_v<T> ? "a number" : "an integer"));
            }
        }
    }

    void list(const std::string& key, std::vector<double>& into)
    {
        if (auto t = text(key)) {
            const std::string where = path_ + "." + key;
            for (const auto& tok : split_csv_line(*t)) {
                try {
                    into.push_back(parse_double(tok, where));
                } catch (const std::invalid_argument&) {
                    bad_config("element " + where + " holds '" + tok + "', expected a number");
                }
            }
        }
    }

    void close() const
    {
        for (const auto& [key, n] : count_)
            if (!claimed_.count(key)) bad_config("unknown element " + path_ + "." + key);
    }

private:
    const XmlElement& el_;
    std::string path_;
    std::map<std::string, int> count_;
    std::set<std::string> claimed_;
};

SimConfig from_document(const XmlElement& root)
{
    if (root.tag != "simulation") bad_config("expected a single <simulation> root element");
    SimConfig c;
    Claim sim(root, "simulation");
    if (const XmlElement* e = sim.single("domain")) {
        Claim d(*e, "simulation.domain");
        d.number("x_min", c.x_min);
        d.number("x_max", c.x_max);
        d.number("y_min", c.y_min);
        d.number("y_max", c.y_max);
        d.number("z_min", c.z_min);
        d.number("z_max", c.z_max);
        d.number("dx", c.dx);
        d.number("dy", c.dy);
        d.number("dz", c.dz);
        d.close();
    }
    if (const XmlElement* e = sim.single("overall")) {
        Claim o(*e, "simulation.overall");
        o.number("max_time", c.max_time);
        o.number("dt_diff", c.dt_diff);
        o.number("dt_mech", c.dt_mech);
        o.number("dt_cell", c.dt_cell);
        o.close();
    }
    if (const XmlElement* e = sim.single("parallel")) {
        Claim p(*e, "simulation.parallel");
        if (auto b = p.text("backend")) {
            if (*b != "serial" && *b != "parallel")
                bad_config("element simulation.parallel.backend holds '" + *b + "', expected 'serial' or 'parallel'");
            c.parallel_backend = *b == "parallel";
        }
        p.number("num_threads", c.num_threads);
        p.close();
    }
    if (const XmlElement* e = sim.single("microenvironment")) {
        Claim m(*e, "simulation.microenvironment");
        for (const XmlElement* sub : m.every("substrate")) {
            Claim s(*sub, "simulation.microenvironment.substrate");
            SubstrateConfig sc;
            if (auto n = s.text("name")) sc.name = *n;
            if (sc.name.empty()) bad_config("element simulation.microenvironment.substrate needs a non-empty <name>");
            s.number("diffusion_coefficient", sc.diffusion_coefficient);
            s.number("decay_rate", sc.decay_rate);
            s.number("initial_condition", sc.initial_condition);
            double dv = 0.0;
            if (s.present("dirichlet_boundary_value")) {
                s.number("dirichlet_boundary_value", dv);
                sc.dirichlet_boundary_value = dv;
            }
            s.close();
            c.substrates.push_back(std::move(sc));
        }
        m.close();
    }
    if (const XmlElement* e = sim.single("agents")) {
        Claim a(*e, "simulation.agents");
        if (auto f = a.text("file")) c.agent_file = *f;
        static const char* inline_keys[] = {"count",   "placement",    "seed",
                                            "volume",  "secretion_rates", "uptake_rates",
                                            "saturation_densities"};
        const bool has_inline = std::any_of(std::begin(inline_keys), std::end(inline_keys),
                                            [&](const char* k) { return a.present(k); });
        if (c.agent_file && has_inline)
            bad_config("element simulation.agents must give either <file> or an inline <count>/<placement> block, "
                       "not both");
        if (has_inline) {
            InlineAgentsConfig ia;
            a.number("count", ia.count);
            if (auto p = a.text("placement")) ia.placement = *p;
            std::int64_t seed = 0;
            if (a.present("seed")) {
                a.number("seed", seed);
                ia.seed = static_cast<std::uint64_t>(seed);
            }
            a.number("volume", ia.volume);
            a.list("secretion_rates", ia.secretion_rates);
            a.list("uptake_rates", ia.uptake_rates);
            a.list("saturation_densities", ia.saturation_densities);
            c.inline_agents = std::move(ia);
        }
        a.close();
    }
    if (const XmlElement* e = sim.single("save")) {
        Claim s(*e, "simulation.save");
        s.number("snapshot_interval", c.snapshot_interval);
        if (auto f = s.text("folder")) c.output_folder = *f;
        s.close();
    }
    sim.close();
    c.validate();
    return c;
}

void require_integral_ratio(double coarse, double fine, const char* what)
{
    const double r = coarse / fine;
    const auto n = static_cast<std::int64_t>(std::llround(r));
    if (n < 1 || std::abs(r - static_cast<double>(n)) > 1e-9 * r)
        bad_config(std::string(what) + " = " + format_double(r) + " must be a positive integer");
}

} // namespace

void SimConfig::validate() const
{
    (void)mesh(); // bounds / spacings
    if (!(dt_diff > 0.0) || !(dt_mech > 0.0) || !(dt_cell > 0.0))
        bad_config("step sizes dt_diff/dt_mech/dt_cell must be positive");
    if (dt_diff > dt_mech || dt_mech > dt_cell) bad_config("step sizes must satisfy dt_diff <= dt_mech <= dt_cell");
    require_integral_ratio(dt_mech, dt_diff, "dt_mech/dt_diff");
    require_integral_ratio(dt_cell, dt_mech, "dt_cell/dt_mech");
    if (max_time < 0.0) bad_config("max_time must be non-negative");
    if (num_threads < 1) bad_config("num_threads must be at least 1");
    if (substrates.empty()) bad_config("at least one substrate must be declared");
    std::set<std::string> seen;
    for (const auto& s : substrates) {
        if (s.name.empty()) bad_config("substrate names must be non-empty");
        if (!seen.insert(s.name).second) bad_config("duplicate substrate name '" + s.name + "'");
        if (s.diffusion_coefficient < 0.0) bad_config("substrate '" + s.name + "' diffusion_coefficient must be >= 0");
        if (s.decay_rate < 0.0) bad_config("substrate '" + s.name + "' decay_rate must be >= 0");
    }
    if (agent_file && inline_agents) bad_config("agents: give either a file or an inline block");
    if (inline_agents) {
        const InlineAgentsConfig& ia = *inline_agents;
        if (ia.count < 0) bad_config("agents.count must be >= 0");
        if (!(ia.volume > 0.0)) bad_config("agents.volume must be positive");
        if (ia.placement != "random" && ia.placement != "center")
            bad_config("agents.placement must be 'random' or 'center', got '" + ia.placement + "'");
        const std::pair<const std::vector<double>*, const char*> lists[] = {
            {&ia.secretion_rates, "secretion_rates"},
            {&ia.uptake_rates, "uptake_rates"},
            {&ia.saturation_densities, "saturation_densities"}};
        for (const auto& [v, name] : lists) {
            if (!v->empty() && v->size() != substrates.size())
                bad_config(std::string("agents.") + name + " must list one value per substrate");
            for (double x : *v)
                if (x < 0.0) bad_config(std::string("agents.") + name + " entries must be >= 0");
        }
    }
}

CartesianMesh SimConfig::mesh() const
{
    return CartesianMesh::from_bounds(x_min, x_max, y_min, y_max, z_min, z_max, dx, dy, dz);
}

SimConfig parse_config_text(const std::string& xml_text)
{
    return from_document(XmlDocument(xml_text, "").read_root());
}

SimConfig parse_config(const std::string& path)
{
    if (!std::filesystem::exists(path)) bad_config("config file not found: " + path);
    std::ifstream in(path, std::ios::binary);
    std::stringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    SimConfig c = from_document(XmlDocument(text, " in " + path).read_root());
    if (c.agent_file && !std::filesystem::exists(*c.agent_file)) bad_config("agent file not found: " + *c.agent_file);
    return c;
}

std::string serialize_config(const SimConfig& c)
{
    std::ostringstream o;
    auto leaf = [&](int depth, const char* key, const std::string& value) {
        o << std::string(static_cast<std::size_t>(2 * depth), ' ') << '<' << key << '>' << value << "</" << key
          << ">\n";
    };
    auto joined = [](const std::vector<double>& v) {
        std::string s;
        for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + format_double(v[i]);
        return s;
    };
    o << "<simulation>\n  <domain>\n";
    leaf(2, "x_min", format_double(c.x_min));
    leaf(2, "x_max", format_double(c.x_max));
    leaf(2, "y_min", format_double(c.y_min));
    leaf(2, "y_max", format_double(c.y_max));
    leaf(2, "z_min", format_double(c.z_min));
    leaf(2, "z_max", format_double(c.z_max));
    leaf(2, "dx", format_double(c.dx));
    leaf(2, "dy", format_double(c.dy));
    leaf(2, "dz", format_double(c.dz));
    o << "  </domain>\n  <overall>\n";
    leaf(2, "max_time", format_double(c.max_time));
    leaf(2, "dt_diff", format_double(c.dt_diff));
    leaf(2, "dt_mech", format_double(c.dt_mech));
    leaf(2, "dt_cell", format_double(c.dt_cell));
    o << "  </overall>\n  <parallel>\n";
    leaf(2, "backend", c.parallel_backend ? "parallel" : "serial");
    leaf(2, "num_threads", format_int(c.num_threads));
    o << "  </parallel>\n  <microenvironment>\n";
    for (const auto& s : c.substrates) {
        o << "    <substrate>\n";
        leaf(3, "name", s.name);
        leaf(3, "diffusion_coefficient", format_double(s.diffusion_coefficient));
        leaf(3, "decay_rate", format_double(s.decay_rate));
        leaf(3, "initial_condition", format_double(s.initial_condition));
        if (s.dirichlet_boundary_value) leaf(3, "dirichlet_boundary_value", format_double(*s.dirichlet_boundary_value));
        o << "    </substrate>\n";
    }
    o << "  </microenvironment>\n";
    if (c.agent_file || c.inline_agents) {
        o << "  <agents>\n";
        if (c.agent_file) leaf(2, "file", *c.agent_file);
        if (const auto& ia = c.inline_agents) {
            leaf(2, "count", format_int(ia->count));
            leaf(2, "placement", ia->placement);
            leaf(2, "seed", format_int(static_cast<std::int64_t>(ia->seed)));
            leaf(2, "volume", format_double(ia->volume));
            if (!ia->secretion_rates.empty()) leaf(2, "secretion_rates", joined(ia->secretion_rates));
            if (!ia->uptake_rates.empty()) leaf(2, "uptake_rates", joined(ia->uptake_rates));
            if (!ia->saturation_densities.empty()) leaf(2, "saturation_densities", joined(ia->saturation_densities));
        }
        o << "  </agents>\n";
    }
    o << "  <save>\n";
    leaf(2, "snapshot_interval", format_double(c.snapshot_interval));
    leaf(2, "folder", c.output_folder);
    o << "  </save>\n</simulation>\n";
    return o.str();
}

void save_config(const SimConfig& config, const std::string& path)
{
    std::ofstream out(path, std::ios::binary);
    if (!out) throw io_error("cannot open " + path + " for writing");
    out << serialize_config(config);
    if (!out) throw io_error("failed writing " + path);
}

Microenvironment build_microenvironment(const SimConfig& config)
{
    config.validate();
    const CartesianMesh mesh = config.mesh();
    std::vector<SubstrateParams> subs;
    for (const auto& s : config.substrates)
        subs.push_back({s.name, s.diffusion_coefficient, s.decay_rate, s.initial_condition});
    Microenvironment env = Microenvironment::create(mesh, std::move(subs));
    const int S = config.substrate_count();
    std::vector<std::uint8_t> mask(static_cast<std::size_t>(S), 0);
    std::vector<double> values(static_cast<std::size_t>(S), 0.0);
    bool clamped = false;
    for (int s = 0; s < S; ++s)
        if (const auto& v = config.substrates[static_cast<std::size_t>(s)].dirichlet_boundary_value) {
            mask[static_cast<std::size_t>(s)] = 1;
            values[static_cast<std::size_t>(s)] = *v;
            clamped = true;
        }
    if (clamped)
        for (int k = 0; k < mesh.nz; ++k)
            for (int j = 0; j < mesh.ny; ++j)
                for (int i = 0; i < mesh.nx; ++i)
                    if (mesh.is_boundary_voxel(i, j, k))
                        env.dirichlet.add(mesh.voxel_index(i, j, k), mask, values, mesh.voxel_count(), S);
    return env;
}

AgentPopulation build_agents(const SimConfig& config, const CartesianMesh& mesh)
{
    const int S = config.substrate_count();
    if (config.agent_file) {
        std::vector<std::string> names;
        for (const auto& s : config.substrates) names.push_back(s.name);
        return load_agents(*config.agent_file, mesh, names);
    }
    if (!config.inline_agents) return {};
    const InlineAgentsConfig& ia = *config.inline_agents;
    auto per_substrate = [&](const std::vector<double>& v) {
        return v.empty() ? std::vector<double>(static_cast<std::size_t>(S), 0.0) : v;
    };
    std::mt19937_64 engine(ia.seed);
    std::uniform_real_distribution<double> along_x(mesh.x_min, mesh.x_max), along_y(mesh.y_min, mesh.y_max),
        along_z(mesh.z_min, mesh.z_max);
    const std::array<double, 3> middle = {(mesh.x_min + mesh.x_max) / 2.0, (mesh.y_min + mesh.y_max) / 2.0,
                                          (mesh.z_min + mesh.z_max) / 2.0};
    std::vector<CellAgent> cells(static_cast<std::size_t>(ia.count));
    for (std::int64_t n = 0; n < ia.count; ++n) {
        CellAgent& a = cells[static_cast<std::size_t>(n)];
        a.id = n;
        a.volume = ia.volume;
        a.secretion_rates = per_substrate(ia.secretion_rates);
        a.uptake_rates = per_substrate(ia.uptake_rates);
        a.saturation_densities = per_substrate(ia.saturation_densities);
        if (ia.placement == "center") {
            a.position = middle;
        } else { // x, y, z drawn in that order
            const double x = along_x(engine);
            const double y = along_y(engine);
            const double z = along_z(engine);
            a.position = {x, y, z};
        }
    }
    return AgentPopulation(std::move(cells), mesh, S);
}

} // namespace biodiff_b200
