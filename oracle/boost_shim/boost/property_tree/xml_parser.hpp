// Test infrastructure only (oracle/): read_xml for the Boost shim (see
// ptree.hpp). Follows Boost's rapidxml-based reader as config.cpp uses it
// (flags trim_whitespace | no_comments): an element becomes a child keyed by
// its tag; attributes go under "<xmlattr>"; text (and CDATA) is appended to
// the element's data, trimmed and with whitespace runs collapsed to one
// space; comments, processing instructions and the declaration are dropped.
// Entities &lt; &gt; &amp; &quot; &apos; &#N; &#xN; are decoded. Errors throw
// xml_parser_error(message, line).
#pragma once

#include "ptree.hpp"

#include <cctype>
#include <fstream>
#include <istream>
#include <iterator>
#include <sstream>
#include <string>

namespace boost {
namespace property_tree {

class xml_parser_error : public std::runtime_error {
public:
    xml_parser_error(const std::string& message, unsigned long line)
        : std::runtime_error(message), message_(message), line_(line)
    {
    }
    const std::string& message() const { return message_; }
    unsigned long line() const { return line_; }

private:
    std::string message_;
    unsigned long line_;
};

namespace xml_parser {

constexpr int no_concat_text = 1;
constexpr int no_comments = 2;
constexpr int trim_whitespace = 4;

namespace shim {

struct Reader {
    const std::string& s;
    std::size_t p = 0;
    int flags = 0;

    unsigned long line_at(std::size_t pos) const
    {
        unsigned long l = 1;
        for (std::size_t i = 0; i < pos && i < s.size(); ++i)
            if (s[i] == '\n') ++l;
        return l;
    }
    [[noreturn]] void error(const std::string& what) const { throw xml_parser_error(what, line_at(p)); }
    bool starts(const char* t) const { return s.compare(p, std::char_traits<char>::length(t), t) == 0; }
    void skip_ws()
    {
        while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    }
    static bool name_char(char c)
    {
        return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.' || c == ':';
    }
    std::string name()
    {
        const std::size_t b = p;
        while (p < s.size() && name_char(s[p])) ++p;
        if (p == b) error("expected element name");
        return s.substr(b, p - b);
    }
    std::string decode(const std::string& raw) const
    {
        std::string out;
        for (std::size_t i = 0; i < raw.size(); ++i) {
            if (raw[i] != '&') {
                out += raw[i];
                continue;
            }
            const std::size_t e = raw.find(';', i);
            if (e == std::string::npos) {
                out += raw[i];
                continue;
            }
            const std::string ent = raw.substr(i + 1, e - i - 1);
            if (ent == "lt") out += '<';
            else if (ent == "gt") out += '>';
            else if (ent == "amp") out += '&';
            else if (ent == "quot") out += '"';
            else if (ent == "apos") out += '\'';
            else if (!ent.empty() && ent[0] == '#') {
                const unsigned long code = ent.size() > 1 && (ent[1] == 'x' || ent[1] == 'X')
                                               ? std::stoul(ent.substr(2), nullptr, 16)
                                               : std::stoul(ent.substr(1), nullptr, 10);
                out += static_cast<char>(code);
            } else {
                out += raw.substr(i, e - i + 1);
            }
            i = e;
        }
        return out;
    }
    std::string normalize(const std::string& t) const
    {
        if (!(flags & trim_whitespace)) return t;
        std::string out;
        bool ws = false;
        for (char c : t) {
            if (std::isspace(static_cast<unsigned char>(c))) {
                ws = true;
                continue;
            }
            if (ws && !out.empty()) out += ' ';
            ws = false;
            out += c;
        }
        return out;
    }
    void misc() // comments, processing instructions, doctype between nodes
    {
        for (;;) {
            skip_ws();
            if (starts("<!--")) {
                const std::size_t e = s.find("-->", p + 4);
                if (e == std::string::npos) error("unexpected end of data");
                p = e + 3;
            } else if (starts("<?")) {
                const std::size_t e = s.find("?>", p + 2);
                if (e == std::string::npos) error("unexpected end of data");
                p = e + 2;
            } else if (starts("<!DOCTYPE")) {
                const std::size_t e = s.find('>', p);
                if (e == std::string::npos) error("unexpected end of data");
                p = e + 1;
            } else {
                return;
            }
        }
    }
    void element(ptree& parent)
    {
        ++p; // '<'
        const std::string tag = name();
        ptree& node = parent.push_back(ptree::value_type(tag, ptree()))->second;
        ptree* attrs = nullptr;
        for (;;) {
            skip_ws();
            if (p >= s.size()) error("unexpected end of data");
            if (s[p] == '/') {
                if (p + 1 >= s.size() || s[p + 1] != '>') error("expected >");
                p += 2;
                return;
            }
            if (s[p] == '>') {
                ++p;
                break;
            }
            const std::string an = name();
            skip_ws();
            if (p >= s.size() || s[p] != '=') error("expected =");
            ++p;
            skip_ws();
            if (p >= s.size() || (s[p] != '"' && s[p] != '\'')) error("expected ' or \"");
            const char q = s[p++];
            const std::size_t e = s.find(q, p);
            if (e == std::string::npos) error("unexpected end of data");
            if (!attrs) attrs = &node.push_back(ptree::value_type("<xmlattr>", ptree()))->second;
            attrs->push_back(ptree::value_type(an, ptree(decode(s.substr(p, e - p)))));
            p = e + 1;
        }
        std::string text;
        for (;;) {
            if (p >= s.size()) error("unexpected end of data");
            if (starts("</")) {
                p += 2;
                const std::string close = name();
                if (close != tag) error("invalid closing tag name");
                skip_ws();
                if (p >= s.size() || s[p] != '>') error("expected >");
                ++p;
                break;
            }
            if (starts("<!--")) {
                const std::size_t e = s.find("-->", p + 4);
                if (e == std::string::npos) error("unexpected end of data");
                if (!(flags & no_comments))
                    node.push_back(ptree::value_type("<xmlcomment>", ptree(s.substr(p + 4, e - p - 4))));
                p = e + 3;
                continue;
            }
            if (starts("<![CDATA[")) {
                const std::size_t e = s.find("]]>", p + 9);
                if (e == std::string::npos) error("unexpected end of data");
                text += s.substr(p + 9, e - p - 9);
                p = e + 3;
                continue;
            }
            if (starts("<?")) {
                const std::size_t e = s.find("?>", p + 2);
                if (e == std::string::npos) error("unexpected end of data");
                p = e + 2;
                continue;
            }
            if (s[p] == '<') {
                element(node);
                continue;
            }
            const std::size_t e = s.find('<', p);
            if (e == std::string::npos) error("unexpected end of data");
            text += decode(s.substr(p, e - p));
            p = e;
        }
        node.data() += normalize(text);
    }
};

inline void read(const std::string& text, ptree& pt, int flags)
{
    ptree result;
    Reader r{text, 0, flags};
    r.misc();
    if (r.p >= text.size() || text[r.p] != '<') r.error("expected <");
    r.element(result);
    r.misc();
    if (r.p != text.size()) r.error("expected end of data");
    pt.swap(result);
}

} // namespace shim

inline void read_xml(std::istream& in, ptree& pt, int flags = 0)
{
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    shim::read(text, pt, flags);
}

inline void read_xml(const std::string& path, ptree& pt, int flags = 0)
{
    std::ifstream in(path, std::ios::binary);
    if (!in) throw xml_parser_error("cannot open file", 0);
    read_xml(in, pt, flags);
}

} // namespace xml_parser

using xml_parser::read_xml;

} // namespace property_tree
} // namespace boost
