// Test infrastructure only (oracle/): the few pieces of Boost.PropertyTree
// the reference's config.cpp uses (config.cpp:6-7, 22, 53-126, 295-323), so
// the reference's own XML config parser compiles here without Boost and can
// serve as the oracle for the product's config ingest. Not a general
// property tree: an ordered list of (key, subtree) children plus a data
// string, get_child / get_value<std::string>, push_back.
#pragma once

#include <list>
#include <stdexcept>
#include <string>
#include <utility>

namespace boost {
namespace property_tree {

struct ptree_bad_path : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class ptree {
public:
    using value_type = std::pair<const std::string, ptree>;
    using container = std::list<value_type>;
    using iterator = container::iterator;
    using const_iterator = container::const_iterator;

    ptree() = default;
    explicit ptree(std::string data) : data_(std::move(data)) {}
    ptree(const ptree&) = default;
    ptree& operator=(const ptree& o) // const keys: rebuild instead of element-wise assignment
    {
        if (this != &o) {
            ptree tmp(o);
            swap(tmp);
        }
        return *this;
    }
    void swap(ptree& o)
    {
        children_.swap(o.children_);
        data_.swap(o.data_);
    }

    const_iterator begin() const { return children_.begin(); }
    const_iterator end() const { return children_.end(); }
    iterator begin() { return children_.begin(); }
    iterator end() { return children_.end(); }

    iterator push_back(const value_type& v) { return children_.insert(children_.end(), v); }

    std::string& data() { return data_; }
    const std::string& data() const { return data_; }

    const ptree& get_child(const std::string& key) const
    {
        for (const auto& c : children_)
            if (c.first == key) return c.second;
        throw ptree_bad_path("No such node (" + key + ")");
    }

    template <class T>
    T get_value() const;

private:
    container children_;
    std::string data_;
};

template <>
inline std::string ptree::get_value<std::string>() const
{
    return data_;
}

} // namespace property_tree
} // namespace boost
